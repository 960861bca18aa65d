"""Diagnostic: what the hottest set's event stream looks like at config 3
(shard 0 of 8) with the models' own decisions -- how many distinct gids per
512-event window, and where the prefetch events fall.  Run under gpurun."""
import sys

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
hp.gids[:n].copy_(torch.from_numpy(t.gid_array.astype(np.int32)))
hp.launch(n)
torch.cuda.synchronize()
K = hp.K
S = C32 // 32
g = t.gid_array
pf = hp.pf[:K].cpu().numpy()
vals, cnt = np.unique(pf, return_counts=True)
o = np.argsort(cnt)[::-1][:10]
print("distinct prefetch ids", len(vals), "top", list(zip(vals[o].tolist(), cnt[o].tolist())))
sets = g % S
hs = np.bincount(sets, minlength=S).argmax()
print("hot set", hs, "serve events", int((sets == hs).sum()))
print("prefetch events into the hot set", int((pf % S == hs).sum()),
      "distinct", np.unique(pf[pf % S == hs]).tolist()[:10])
# the hot set's stream, chunk by chunk: S events, last-U per gid, P events
ev = []
gk = g[:K * 15].reshape(K, 15)
for k in range(min(K, 400_000)):
    row = gk[k]
    m = row % S == hs
    ev.extend(row[m].tolist())
    seen = set()
    for x in row[::-1][(row[::-1] % S) == hs]:
        if x not in seen:
            seen.add(x)
            ev.append(int(x))
    ev.extend([int(x) for x in pf[k] if x % S == hs])
ev = np.asarray(ev)
W = 512
d = [len(np.unique(ev[i:i + W])) for i in range(0, len(ev) - W, W)]
h = np.bincount(np.minimum(d, 9))
print("windows", len(d), "distinct-gid histogram (1..8, 9+):", h[1:].tolist())
