"""Diagnostic: timeline of one HotPath step at config 2 (event timestamps
relative to the step start, per pipeline piece) -- where the tail after the
last forward comes from.  Run under gpurun."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_08568_b200 as rb  # noqa: E402
from paper_2511_08568_b200.model import DeviceModel, init_params_device  # noqa: E402
from paper_2511_08568_b200.pipeline import HotPath  # noqa: E402

pieces = int(sys.argv[1]) if len(sys.argv) > 1 else 8
model_sms = int(sys.argv[2]) if len(sys.argv) > 2 else 146
with_lru = not (len(sys.argv) > 3 and sys.argv[3] == "nolru")
t = rb.generate_trace(rb.TraceGenConfig([50_000] * 256, 25_000_000, 1.05, 0.4, 32, 2))
C = int(0.2 * t.unique_count)
C32 = C - C % 32
cp, ec = init_params_device("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
pp, ep = init_params_device("prefetch", t.table_sizes, dim=64, seed=1, init_scale=0.4)
n = len(t)
hp = HotPath(DeviceModel(cp, ec), DeviceModel(pp, ep), t.table_sizes, C32, n, ways=32,
             lru_capacity=C32 if with_lru else None, lru_ways=32, pieces=pieces,
             model_sms=model_sms)
hp.gids[:n].copy_(torch.from_numpy(t.gid_array.astype(np.int32)))
for _ in range(3):
    hp.launch(n)
torch.cuda.synchronize()
hp.enable_stage_timing(True)
start = torch.cuda.Event(enable_timing=True)
start.record()
hp.launch(n)
end = torch.cuda.Event(enable_timing=True)
end.record()
torch.cuda.synchronize()
print(f"step {start.elapsed_time(end):.1f} ms")
ev = hp.events
for key in ("caching_fwd", "prefetch_fwd", "replay", "lru", "tail"):
    xs = ev.get(key, [])
    spans = [(start.elapsed_time(xs[i]), start.elapsed_time(xs[i + 1]))
             for i in range(0, len(xs) - 1, 2)]
    print(key, " ".join(f"[{a:.1f},{b:.1f}]" for a, b in spans))
