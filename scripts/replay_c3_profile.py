"""Diagnostic: where the config-3 (shard 0 of 8) replay time goes.  Builds the
shard's state, scores the trace once (HotPath), then times the whole-trace
replay (one launch, idle GPU) and the per-piece replays, and counts the
hottest set's events by type after the event builder's collapsing.  Run under
gpurun; prints only diagnostics."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2511_08568_b200.model import DeviceModel  # noqa: E402
from paper_2511_08568_b200.pipeline import HotPath  # noqa: E402


class A:
    accesses, tables, rows, dim, init_scale = 500_000_000, 856, 100_000, 64, 0.4
    shards_eff, world, shard_index = 8, 1, 0


t, U, C, C32, cp, emb_c, pp, emb_p, _, sh = bench.build_state_config3(A, 0, torch)
n = len(t)
hp = HotPath(DeviceModel(cp, emb_c, decode_ids=sh.total_ids),
             DeviceModel(pp, emb_p, decode_ids=sh.total_ids), t.table_sizes, C32, n,
             ways=32, lru_capacity=C32, lru_ways=32, shard=sh, model_sms=124)
del emb_c, emb_p
hp.gids[:n].copy_(torch.from_numpy(t.gid_array.astype(np.int32)))
for _ in range(2):
    hp.launch(n)
torch.cuda.synchronize()
K = hp.K
S = C32 // 32
print(f"n={n} K={K} U={U} C32={C32} S={S}")


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


g = hp.gids[:n]
bits, pf = hp.bits[:K], hp.pf[:K]
buf = hp.buffer


def whole():
    buf.reset()
    buf.run(g, bits, pf)


print(f"whole-trace replay, one launch: {timed(whole):.2f} ms")
lru = hp.lru


def lru_run():
    lru.reset()
    lru.run(g)


print(f"whole-trace LRU, one launch: {timed(lru_run):.2f} ms")
hp.enable_stage_timing(True)
hp.launch(n)
torch.cuda.synchronize()
print("pipelined stages", {k: round(v, 2) for k, v in hp.stage_times().items()})
ev = hp.events["replay"]
print("replay pieces ms", [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(0, len(ev), 2)])

# the hottest set's event stream (build_events_kernel's collapsing restated)
ga = t.gid_array.astype(np.int64)
sets = ga % S
hs = int(np.bincount(sets, minlength=S).argmax())
b = bits.cpu().numpy()
p = pf.cpu().numpy().astype(np.int64)
nS = nU = nP = 0
runs = 0
last_g = -1
changes = 0
t0 = time.time()
kin = ga[:K * 15].reshape(K, 15)
m = (kin % S) == hs
for k in np.nonzero(m.any(axis=1))[0]:
    row = kin[k]
    prev = None
    for i in range(15):
        if row[i] % S != hs:
            continue
        if row[i] != prev:
            nS += 1
            if row[i] != last_g:
                changes += 1
                last_g = row[i]
        prev = row[i]
    seen = set()
    for i in range(14, -1, -1):
        if row[i] % S == hs and row[i] not in seen:
            seen.add(row[i])
            nU += 1
            if row[i] != last_g:
                changes += 1
                last_g = row[i]
    for q in p[k]:
        if q >= 0 and q % S == hs:
            nP += 1
            if q != last_g:
                changes += 1
                last_g = q
print(f"hot set {hs}: accesses {int((sets == hs).sum())}, events S {nS} U {nU} P {nP}, "
      f"gid changes along the stream {changes} ({time.time() - t0:.0f}s to count)")
top = np.bincount(ga).argmax()
print(f"top id {top} accesses {int((ga == top).sum())} set {top % S}")
