"""Config-5 sweep (BASELINE.json configs[4]): buffer 5-40% of unique rows and
evaluation window 5-30 accesses, RecMG's learned buffer vs 32-way LRU / LFU
and the offline optimum — the paper's §VII comparisons
on the GPU engine.

    python -m paper_2511_08568_b200.sweep --accesses 1000000 --out sweep.json
"""
from __future__ import annotations

import argparse
import json
import math
import time

from . import _native
from .cache_sim import CacheConfig, Policy, simulate
from .model import init_params
from .pipeline import HotPath
from .runtime import correctness_vs_window
from .trace import TraceGenConfig, generate_trace

FRACTIONS = (0.05, 0.10, 0.15, 0.20, 0.30, 0.40)
RATIOS = (1, 2, 3, 4, 5, 6)   # eval window = ratio * l_out = 5..30


def run(trace, cparams, pparams, fractions=FRACTIONS, ratios=RATIOS, ways=32):
    U = trace.unique_count
    torch = _native.torch_cuda()
    rows = []
    g = torch.from_numpy(trace.gid_array.astype("int32")).pin_memory()
    for f in fractions:
        C = int(math.floor(f * U))
        C -= C % ways
        if C < ways:
            continue
        hp = HotPath(cparams, pparams, trace.table_sizes, C, len(trace), ways=ways,
                     lru_capacity=C, lru_ways=ways)
        rep, (lh, lm) = hp.replay_host(g)
        lfu = simulate(trace, CacheConfig(C, Policy.LFU, ways), per_access=False)
        opt = simulate(trace, CacheConfig(C, Policy.OPTGEN, ways), per_access=False)
        rows.append({"fraction": f, "capacity": C, "recmg_on_demand": rep.on_demand,
                     "recmg_hits": rep.hits, "recmg_prefetch_hits": rep.prefetch_hits,
                     "lru32_misses": lm, "lfu32_misses": lfu.misses, "optgen32_misses": opt.misses,
                     "on_demand_vs_lru32": rep.on_demand / lm if lm else None})
    windows = correctness_vs_window(trace, pparams, list(ratios))
    return {"unique": U, "capacity_rows": rows,
            "prefetch_correctness_vs_window": {str(r * pparams.l_out): v
                                               for r, v in windows.items()}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--accesses", type=int, default=1_000_000)
    ap.add_argument("--tables", type=int, default=8)
    ap.add_argument("--rows", type=int, default=2000)
    ap.add_argument("--init-scale", type=float, default=0.4)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    t0 = time.time()
    t = generate_trace(TraceGenConfig([a.rows] * a.tables, a.accesses, 1.05, 0.4, 32, 0))
    cp = init_params("caching", t.table_sizes, dim=64, seed=0, init_scale=a.init_scale)
    pp = init_params("prefetch", t.table_sizes, dim=64, seed=1, init_scale=a.init_scale)
    res = run(t, cp, pp)
    res["config"] = {"tables": a.tables, "rows_per_table": a.rows, "accesses": a.accesses,
                     "init_scale": a.init_scale, "models": "random init (no trained checkpoint)",
                     "seconds": time.time() - t0}
    text = json.dumps(res, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    print(text)


if __name__ == "__main__":
    main()
