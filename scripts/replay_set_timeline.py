"""Diagnostic: per-set timeline of the whole-trace replay (and the LRU) at
config 2 -- start / end (globaltimer) and path of every set's warp
(recmg_diag_set_timing), for RECMG_REPLAY_REGS=0 and 1.  Prints the span,
the sets that end last (their length, start, duration), ns per event by path
and set-length bucket.  Run under gpurun."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_08568_b200 as rb  # noqa: E402
from paper_2511_08568_b200 import _native  # noqa: E402
from paper_2511_08568_b200.model import DeviceModel, init_params_device  # noqa: E402
from paper_2511_08568_b200.pipeline import HotPath  # noqa: E402

t = rb.generate_trace(rb.TraceGenConfig([50_000] * 256, 25_000_000, 1.05, 0.4, 32, 2))
C = int(0.2 * t.unique_count)
C32 = C - C % 32
S = C32 // 32
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
L = _native.lib()
L.recmg_diag_set_timing.argtypes = [ctypes.c_void_p]
rec = torch.zeros(8 * S, dtype=torch.int64, device="cuda")


def report(name, r):
    r = r[:4 * S].reshape(S, 4)
    st, en, path, ln, ms = r[:, 0], r[:, 1], r[:, 2] >> 32, r[:, 3] & 0xFFFFFFFF, r[:, 3] >> 32
    ok = en > 0
    t0 = st[ok].min()
    span = (en[ok].max() - t0) / 1e6
    print(f"== {name}: span {span:.2f} ms over {ok.sum()} sets")
    last = np.argsort(-en)[:12]
    for s_ in last:
        print(f"   set {s_:6d} path {path[s_]} sm {r[s_, 2] & 0xFFFFFFFF:3d} len {ln[s_]:8d} start {(st[s_]-t0)/1e6:7.3f} "
              f"dur {(en[s_]-st[s_])/1e6:7.3f} ms  {(en[s_]-st[s_])/max(ln[s_],1):6.1f} ns/ev, "
              f"misses {ms[s_]} ({ms[s_]/max(ln[s_],1):.2f}/ev)")
    for p_ in (0, 1):
        for lo_, hi_ in ((0, 2048), (2048, 8192), (8192, 32768), (32768, 1 << 40)):
            m = ok & (path == p_) & (ln >= lo_) & (ln < hi_)
            if m.sum():
                d = (en[m] - st[m]).astype(np.float64)
                print(f"   path {p_} len [{lo_}, {hi_}): {m.sum():5d} sets, "
                      f"{d.sum() / ln[m].sum():6.1f} ns/event, max dur {d.max() / 1e6:.3f} ms")


from paper_2511_08568_b200.engine import LruSim  # noqa: E402
lru = LruSim(C32, t.total_ids if hasattr(t, "total_ids") else sum(t.table_sizes), 32, n)
for _ in range(2):
    rec.zero_()
    L.recmg_diag_set_timing(rec.data_ptr())
    buf.reset()
    lru.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    assert buf.run_chunks_lru(g, 0, K, True, lru, bits, pf, skip_stats=True)
    e1.record()
    torch.cuda.synchronize()
print(f"fused replay + LRU (events + partition + both): {e0.elapsed_time(e1):.2f} ms")
r = rec.cpu().numpy()
both = np.concatenate([r[:4 * S].reshape(S, 4), r[4 * S:].reshape(S, 4)])
t0 = both[:, 0][both[:, 1] > 0].min()
report("fused: priority replay items", r[:4 * S])
rr = r[4 * S:].copy()
report("fused: LRU items", rr)
L.recmg_diag_set_timing(None)
if os.environ.get("TIMELINE_ONLY_HEAVY"):
    os.environ["RECMG_REPLAY_ONLY_HEAVY"] = "1"
    for fused in (True, False):
        rec.zero_()
        L.recmg_diag_set_timing(rec.data_ptr())
        buf.reset()
        lru.reset()
        if fused:
            assert buf.run_chunks_lru(g, 0, K, True, lru, bits, pf, skip_stats=True)
        else:
            buf.run_chunks(g, 0, K, True, bits, pf, skip_stats=True)
        torch.cuda.synchronize()
        r = rec.cpu().numpy()
        report(f"heavy only, fused={fused}: priority items", r[:4 * S])
        if fused:
            report("heavy only, fused: LRU items", r[4 * S:].copy())
    L.recmg_diag_set_timing(None)
    os.environ.pop("RECMG_REPLAY_ONLY_HEAVY")

for regs, queue in ():
    os.environ["RECMG_REPLAY_REGS"] = regs
    os.environ["RECMG_REPLAY_QUEUE"] = queue
    for _ in range(2):
        rec.zero_()
        L.recmg_diag_set_timing(rec.data_ptr())
        buf.reset()
        buf.run_chunks(g, 0, K, True, bits, pf, skip_stats=True)
        torch.cuda.synchronize()
    report(f"replay regs={regs} queue={queue}", rec.cpu().numpy())
    rec.zero_()
    hp.lru.reset()
    hp.lru.run(g)
    torch.cuda.synchronize()
    report(f"lru regs={regs} queue={queue}", rec.cpu().numpy())
    L.recmg_diag_set_timing(None)
