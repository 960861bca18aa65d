"""Diagnostic: one replay piece (recmg_replay_chunks) alone on the full GPU,
beside a memory-silent SM hog that leaves it 12 SMs, and beside the real
caching forward on 136 SMs -- separates SM starvation from memory-system
interference.  Run under gpurun after nvcc-ing scripts/sm_hog.cu."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_08568_b200 as rb  # noqa: E402
from paper_2511_08568_b200 import _native  # noqa: E402
from paper_2511_08568_b200.model import DeviceModel, init_params_device  # noqa: E402
from paper_2511_08568_b200.pipeline import HotPath  # noqa: E402

hog = ctypes.CDLL("scripts/libsmhog.so")
hog.sm_hog.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
hog.shape_hog.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_void_p]
hog.gather_hog.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_longlong, ctypes.c_void_p]
hog.mem_hog.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_longlong, ctypes.c_void_p]
t = rb.generate_trace(rb.TraceGenConfig([50_000] * 256, 25_000_000, 1.05, 0.4, 32, 2))
C = int(0.2 * t.unique_count)
C32 = C - C % 32
cp, ec = init_params_device("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
pp, ep = init_params_device("prefetch", t.table_sizes, dim=64, seed=1, init_scale=0.4)
n = len(t)
hp = HotPath(DeviceModel(cp, ec), DeviceModel(pp, ep), t.table_sizes, C32, n, ways=32,
             lru_capacity=None, pieces=8, model_sms=136)
hp.gids[:n].copy_(torch.from_numpy(t.gid_array.astype(np.int32)))
hp.launch(n)
torch.cuda.synchronize()
K = hp.K
pieces = hp._piece_bounds(K)
g = hp.gids[:n]
bits, pf = hp.bits[:K], hp.pf[:K]
side = torch.cuda.Stream()


def replay_pieces(upto, stream):
    """reset + replay pieces [0, upto) on `stream`; returns (start, end) events."""
    with torch.cuda.stream(stream):
        hp.buffer.reset()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for i in range(upto):
            k0, k1 = pieces[i]
            hp.buffer.run_chunks(g, k0, k1, i == len(pieces) - 1, bits, pf)
        e.record(stream)
    return s, e


for label in ("alone", "shape136"):
    for rep in range(2):
        torch.cuda.synchronize()
        if label == "hog136":
            hog.sm_hog(136, 300.0, _native.stream_handle(torch))
        elif label == "dram136":
            hog.mem_hog(136, 300.0, 4 << 30, _native.stream_handle(torch))
        elif label == "l2hog136":
            hog.mem_hog(136, 300.0, 64 << 20, _native.stream_handle(torch))
        elif label == "gather136":
            hog.gather_hog(136, 300.0, 12 << 30, _native.stream_handle(torch))
        elif label == "gather136_l2":
            hog.gather_hog(136, 300.0, 64 << 20, _native.stream_handle(torch))
        elif label.startswith("shape"):
            hog.shape_hog(136, 300.0, 1 if "tmem" in label else 0, _native.stream_handle(torch))
        elif label.startswith("caching") or label.startswith("prefetch"):
            L = _native.lib()
            sms = 100 if "100" in label else 136
            prev = L.recmg_set_model_sm_budget(sms)
            gk = hp.gids[:K * 15].view(K, 15)
            tk = hp.tid[:K * 15].view(K, 15)
            for _ in range(4):
                if label.startswith("caching"):
                    hp.caching.forward(gk, tk, logits=hp.clog[:K], bits=hp.bits[:K])
                else:
                    hp.prefetch.forward(gk, tk, logits=hp.plog[:K], pf_gid=hp.pf[:K])
            L.recmg_set_model_sm_budget(prev)
        s, e = replay_pieces(2, side)
        torch.cuda.synchronize()
        print(f"{label}: 2 replay pieces {s.elapsed_time(e):.2f} ms")
