"""Per-CUDA-source-line instruction counts of one kernel from an ncu report (development aid).

    python tools/src_lines.py <report.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
f = None
hdr = None
acc = {}
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or not r[0]:
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        e = int(d["Instructions Executed"] or 0)
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    except (KeyError, ValueError):
        continue
    acc[(f, int(r[0]))] = (e, s, r[1][:90])
tot = sum(v[0] for v in acc.values()) or 1
ts = sum(v[1] for v in acc.values()) or 1
print(f"total warp-instructions {tot}")
for (fn, ln), (e, s, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{fn:14s}{ln:5d} {e / tot * 100:5.1f}% st{s / ts * 100:5.1f}%  {src}")
