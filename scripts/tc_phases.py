"""Per-phase cycle breakdown of the tcgen05 LSTM forwards (diagnostic build,
recmg_model_forward_profile).  Run under gpurun; prints the share of thread
0's timeline per phase, averaged over CTAs."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_08568_b200 as rb
from paper_2511_08568_b200 import _native
from paper_2511_08568_b200.model import DeviceModel, init_params_device

PF_NAMES = {1: "enc Wh0 swap wait+L0 MMA", 2: "enc cell0", 15: "enc Wx1 swap wait", 14: "enc sync",
            12: "enc L1 issue+row prefetch", 13: "enc Q wait+keys", 10: "enc L1 MMA wait",
            11: "enc cell1 / dec L1 cell"}
NAMES = ["enc table init+sync", "enc MMA wait", "enc epilogue", "dec init+sync",
         "dec MMA1 wait", "dec head+scores+sync", "dec softmax/ctx+sync", "dec MMA2 wait",
         "dec cell", "weight loads", "pf L1 MMA wait", "pf L1 cell", "enc MMA issue", "enc row prefetch", "", "other"]

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
t = rb.generate_trace(rb.TraceGenConfig([rows] * 256, n, 1.05, 0.4, 32, 2))
K = rb.num_chunks(len(t))
g = torch.from_numpy(t.gid_array[:K * 15].astype(np.int32).reshape(K, 15)).cuda()
for kind, seed in (("caching", 0), ("prefetch", 1)):
    p, emb = init_params_device(kind, t.table_sizes, dim=64, seed=seed, init_scale=0.4)
    dm = DeviceModel(p, emb)
    tid = dm.table_ids(g)
    out = torch.empty((K, dm.out_len), dtype=torch.float32, device="cuda")
    ws = dm.workspace(K)
    prof = torch.zeros((148, 16), dtype=torch.int64, device="cuda")
    L = _native.lib()
    for it in range(2):
        prof.zero_()
        s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        _native.check(L.recmg_model_forward_profile(ctypes.byref(dm.shape), _native.ptr(dm.packed),
                                                    _native.ptr(g), _native.ptr(tid), K,
                                                    _native.ptr(out), _native.ptr(ws), ws.numel(),
                                                    _native.ptr(prof), _native.stream_handle(torch)))
        s1.record()
        torch.cuda.synchronize()
    pr = prof.cpu().numpy().astype(np.float64)
    tot = pr.sum(axis=1).mean()
    print(f"{kind}: {s0.elapsed_time(s1):.2f} ms, {tot / 1.9e6:.2f} ms of cycles per CTA @1.9GHz")
    for i in range(16):
        v = pr[:, i].mean()
        if v > 0:
            name = PF_NAMES.get(i, NAMES[i]) if kind == "prefetch" else NAMES[i]
            print(f"   {name:26s} {v / tot * 100:5.1f}%")
    del dm, emb
