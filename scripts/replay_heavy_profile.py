"""Diagnostic: the config-2 replay of the heavy list alone (the 32 longest
sets, RECMG_REPLAY_ONLY_HEAVY=1), after one HotPath launch -- the third
replay_smem_kernel launch of this script -- for an ncu --set full capture of
the chain-bound phase (ncu -k regex:replay_smem_kernel -s 2 -c 1).  Run
under gpurun."""
import os
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
os.environ["RECMG_REPLAY_ONLY_HEAVY"] = "1"
for _ in range(3):
    hp.buffer.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hp.buffer.run_chunks(hp.gids[:n], 0, K, True, hp.bits[:K], hp.pf[:K], skip_stats=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"heavy-only replay (events + partition + 32 longest sets): {e0.elapsed_time(e1):.2f} ms")
