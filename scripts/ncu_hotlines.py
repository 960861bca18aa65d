"""Warp-stall samples of one ncu --set full capture, aggregated per source
line (diagnostic).  The SASS page of the capture gives samples per
instruction address; nvdisasm -g of the same build gives each instruction's
file:line, matched by offset from the function start (the opcodes are
checked to agree, so a capture of another build is rejected).

    python scripts/ncu_hotlines.py gpurun_out/prof_0.ncu-rep 'lstm_tc_kernelILi0ELi0E' [top]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda/bin"
rep, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
unit = sys.argv[4] if len(sys.argv) > 4 else "lstm_tc"   # the .cu whose cubin holds fn

csv_text = subprocess.run([f"{CUDA}/ncu", "-i", rep, "--page", "source", "--csv",
                           "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(csv_text)))
hdr, data = rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
key = "Warp Stall Sampling (All Samples)"
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]

with tempfile.TemporaryDirectory() as d:
    subprocess.run([f"{CUDA}/cuobjdump", "-xelf", "all",
                    os.path.join(ROOT, "paper_2511_08568_b200", "librecmg.so")],
                   cwd=d, capture_output=True)
    cubin = os.path.join(d, f"{unit}.sm_100a.cubin")
    sass = subprocess.run([f"{CUDA}/nvdisasm", "-g", "-c", cubin], capture_output=True,
                          text=True).stdout.split("\n")
start = next(i for i, l in enumerate(sass) if l.startswith(".text.") and fn in l)
where, cur = {}, None
for l in sass[start + 1:]:
    if l.startswith(".text.") or l.strip().startswith(".section"):
        break
    m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
    if m:
        where[int(m.group(1), 16)] = (cur, m.group(2))

base = int(data[0][idx["Address"]], 16)
total = sum(float(r[idx[key]] or 0) for r in data)
agg, reasons = {}, {}
for r in data:
    off = int(r[idx["Address"]], 16) - base
    loc, ins = where[off]
    got = r[idx["Source"]].split()
    want = ins.split()
    op = lambda t: t[1] if t[0].startswith("@") else t[0]
    if op(got) != op(want):
        raise SystemExit(f"capture does not match this build at +{off:#x}: {got} vs {want}")
    agg[loc] = agg.get(loc, 0.0) + float(r[idx[key]] or 0)
    for h in stalls:
        reasons.setdefault(loc, {}).setdefault(h, 0.0)
        reasons[loc][h] += float(r[idx[h]] or 0)

src = {}
for f in ("lstm_tc.cu", "umma.cuh", "replay.cu", "partition.cu", "capi.cu"):
    src[f] = open(os.path.join(ROOT, "paper_2511_08568_b200", "csrc", f)).read().split("\n")
print(f"{os.path.basename(rep)} {fn}: {int(total)} warp-stall samples")
for loc, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    f, ln = loc
    main = max(reasons[loc].items(), key=lambda x: x[1])[0][6:]
    text = src[f][ln - 1].strip()[:90] if f in src else ""
    print(f"{100 * v / total:5.2f}%  {main:14s} {f}:{ln:<5d} {text}")
