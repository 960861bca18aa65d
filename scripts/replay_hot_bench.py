"""Diagnostic: per-event cost of the replay kernels (K3 / K4) on a set whose
segment is one long run of a single gid (the config-3 hot set), and on a
Zipf-like mix.  Run under gpurun; prints ms and ns per event."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_08568_b200.engine import BufferReplay, LruSim   # noqa: E402
from paper_2511_08568_b200.trace import num_chunks              # noqa: E402


def timed(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


rng = np.random.default_rng(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
cases = {
    "single gid, 1 set": (np.full(n, 5, np.int32), 100, 32),
    "hot 50% + uniform 1M ids, 1000 sets": (
        np.where(rng.random(n) < 0.5, 7, rng.integers(0, 1_000_000, n)).astype(np.int32),
        1_000_000, 32 * 1000),
}
for name, (g, V, cap) in cases.items():
    gd = torch.from_numpy(g).cuda()
    K = num_chunks(n)
    bits = torch.zeros((K, 15), dtype=torch.uint8, device="cuda")
    pf = torch.from_numpy(rng.integers(0, V, (K, 5)).astype(np.int32)).cuda()
    lru = LruSim(cap, V, 32, n)

    def run_lru():
        lru.reset()
        lru.run(gd)
    t = timed(run_lru)
    hot = int((g % (cap // 32) == g[0] % (cap // 32)).sum())
    print(f"{name}: LRU {t:.2f} ms, {t * 1e6 / hot:.2f} ns per hot-set event ({hot} events)")
    br = BufferReplay(cap, V, 4, 32, n, pf_stride=5)

    def run_rep():
        br.reset()
        br.run(gd, bits, pf)
    t = timed(run_rep)
    print(f"{name}: replay {t:.2f} ms, {t * 1e6 / (hot * 16 / 15):.2f} ns per hot-set event")
