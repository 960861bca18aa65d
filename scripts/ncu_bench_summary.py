"""profiles/ncu_summary.json (read by bench.py for roofline.traffic) from a
round's ncu summary (scripts/ncu_summary.py output): per-launch DRAM bytes
and pipe utilisations of the four captured kernels.

    python scripts/ncu_bench_summary.py profiles/r01h_config2.json "<note>"
"""
import json
import os
import sys

src = sys.argv[1]
note = sys.argv[2] if len(sys.argv) > 2 else ""
d = json.load(open(src))
UNIT = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
TIME = {"s": 1e3, "ms": 1.0, "us": 1e-3, "ns": 1e-6}


def qty(s, table):
    v, u = s.split()
    return float(v) * table[u]


out = {"source": f"{src} (ncu --set full --clock-control none, config 2, 25M accesses, "
                 "8 pipeline pieces: one forward / replay launch = 1/8 of the trace; "
                 f"scripts/ncu_round.sh) {note}".strip()}
for f, name in (("prof_0.ncu-rep", "caching_fwd"), ("prof_1.ncu-rep", "prefetch_fwd"),
                ("prof_2.ncu-rep", "replay"), ("prof_3.ncu-rep", "lru")):
    c = d["captures"][f][0]
    rd, wr = qty(c["dram__bytes_read.sum"], UNIT), qty(c["dram__bytes_write.sum"], UNIT)
    out[name] = {
        "kernel": c["kernel"],
        "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
        "ncu_duration_ms": qty(c["gpu__time_duration.sum"], TIME),
        "tensor_pipe_pct": c["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"],
        "xu_pipe_pct": c["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"],
        "fma_pipe_pct": c["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"],
        "l1tex_throughput_pct": c["l1tex__throughput.avg.pct_of_peak_sustained_active"],
        "warps_active_pct": c["sm__warps_active.avg.pct_of_peak_sustained_active"],
        "registers": c["launch__registers_per_thread"], "grid": c["launch__grid_size"],
        "block": c["launch__block_size"]}
    print(name, round(out[name]["ncu_duration_ms"], 3), "ms",
          round(out[name]["dram_bytes_per_launch"] / 1e9, 3), "GB",
          "XU", out[name]["xu_pipe_pct"], "tensor", out[name]["tensor_pipe_pct"])
dst = os.path.join(os.path.dirname(os.path.abspath(src)), "ncu_summary.json")
json.dump(out, open(dst, "w"), indent=1)
