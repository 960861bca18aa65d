"""Timing of the production tcgen05 forwards (diagnostic): median over reps of
DeviceModel.forward on a config-2-like batch, CUDA events on the current
stream.  Used with scripts/ab.sh for A/B builds (RECMG_LIB)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_08568_b200 as rb
from paper_2511_08568_b200.model import DeviceModel, init_params_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
precision = sys.argv[3] if len(sys.argv) > 3 else "auto"
t = rb.generate_trace(rb.TraceGenConfig([50000] * 256, n, 1.05, 0.4, 32, 2))
K = rb.num_chunks(len(t))
g = torch.from_numpy(t.gid_array[:K * 15].astype(np.int32).reshape(K, 15)).cuda()
import os
if os.environ.get("FWD_IDS") == "const":      # every token the same id: rows always L1 hits
    g.fill_(12345)
elif os.environ.get("FWD_IDS") == "few":      # 64 distinct ids
    g.remainder_(64)
for kind, seed in (("caching", 0), ("prefetch", 1)):
    p, emb = init_params_device(kind, t.table_sizes, dim=64, seed=seed, init_scale=0.4)
    dm = DeviceModel(p, emb, precision=precision)
    tid = dm.table_ids(g)
    out = torch.empty((K, dm.out_len), dtype=torch.float32, device="cuda")
    ms = []
    for it in range(reps + 1):
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        dm.forward(g, tid, logits=out)
        s1.record()
        torch.cuda.synchronize()
        if it:
            ms.append(s0.elapsed_time(s1))
    chk = float(out.double().sum())
    print(f"{kind}: median {np.median(ms):.3f} ms min {min(ms):.3f} ms (K={K}) checksum {chk:.6e}")
