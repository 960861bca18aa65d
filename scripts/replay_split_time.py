"""Diagnostic: whole-trace replay time at config 2 on an idle GPU (one launch,
the decisions of one HotPath pass) -- run with RECMG_LIB set to the
RECMG_DIAG_SETS=1/2 builds to time the heavy sets' chains / the other sets
alone.  Run under gpurun."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_08568_b200 as rb  # noqa: E402
from paper_2511_08568_b200.model import DeviceModel, init_params_device  # noqa: E402
from paper_2511_08568_b200.pipeline import HotPath  # noqa: E402

t = rb.generate_trace(rb.TraceGenConfig([50_000] * 256, 25_000_000, 1.05, 0.4, 32, 2))
C = int(0.2 * t.unique_count)
C32 = C - C % 32
cp, ec = init_params_device("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
pp, ep = init_params_device("prefetch", t.table_sizes, dim=64, seed=1, init_scale=0.4)
n = len(t)
hp = HotPath(DeviceModel(cp, ec), DeviceModel(pp, ep), t.table_sizes, C32, n, ways=32,
             lru_capacity=C32)
hp.gids[:n].copy_(torch.from_numpy(t.gid_array.astype(np.int32)))
hp.launch(n)
torch.cuda.synchronize()
K = hp.K
g, bits, pf = hp.gids[:n], hp.bits[:K], hp.pf[:K]
buf = hp.buffer
import os
for regs, queue in (("0", "1"), ("1", "1"), ("-1", "1")):
    os.environ["RECMG_REPLAY_REGS"] = regs
    os.environ["RECMG_REPLAY_QUEUE"] = queue
    ms, ml = [], []
    for _ in range(7):
        buf.reset()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        buf.run_chunks(g, 0, K, True, bits, pf, skip_stats=True)
        e1.record()
        hp.lru.reset()
        hp.lru.run(g)
        e2.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        ml.append(e1.elapsed_time(e2))
    print(f"RECMG_REPLAY_REGS={regs} QUEUE={queue}: whole-trace replay (events + partition + replay): "
          f"{np.median(ms[1:]):.2f} ms, LRU {np.median(ml[1:]):.2f} ms")
    print("   counters", buf.result(with_coverage=False), "lru", hp.lru.result())
