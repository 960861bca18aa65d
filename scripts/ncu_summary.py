"""Summarise ncu outputs into profiles/: launch-list shares and the key
counters of each --set full capture.  Usage:
    python scripts/ncu_summary.py <tag> gpurun_out/launches.csv gpurun_out/prof_*.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((d["Kernel Name"].split("(")[0], float(d["Metric Value"])))
    tot = sum(t for _, t in out)
    agg = {}
    for k, t in out:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    return {"total_ns": tot, "kernels": {k: {"launches": c, "ns": t, "share": t / tot}
                                         for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])}}


def capture(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{row[i]} {units[i]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    tag = sys.argv[1]
    out = {"tag": tag}
    for p in sys.argv[2:]:
        if p.endswith(".csv"):
            out["launch_list"] = launches(p)
        elif p.endswith(".ncu-rep"):
            out.setdefault("captures", {})[os.path.basename(p)] = capture(p)
    os.makedirs("profiles", exist_ok=True)
    with open(f"profiles/{tag}.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:3000])
