"""Opcode mix and hot regions of one kernel from an ncu report (development aid).

    python tools/sass_mix.py <report.ncu-rep> [kernel-regex]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2:
    args += ["-k", sys.argv[2]]
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
isrc, iss, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(int(r[ie]) for r in data) or 1
ts = sum(int(r[iss]) for r in data) or 1
ops = collections.Counter()
stl = collections.Counter()
for r in data:
    op = r[isrc].split()[0] if r[isrc].split() else "?"
    if op.startswith("@"):
        op = r[isrc].split()[1]
    op = op.split(".")[0]
    ops[op] += int(r[ie])
    stl[op] += int(r[iss])
print(f"total warp-instructions {tot}, stall samples {ts}")
for op, n in ops.most_common(25):
    print(f"  {op:10s} {n / tot * 100:5.1f}%  stalls {stl[op] / ts * 100:5.1f}%")
# hot regions: windows of 32 SASS lines
W = 32
reg = []
for k in range(0, len(data), W):
    e = sum(int(r[ie]) for r in data[k:k + W])
    s = sum(int(r[iss]) for r in data[k:k + W])
    reg.append((e, s, k))
print("hot 32-instruction windows (line, inst %, stall %):")
for e, s, k in sorted(reg, reverse=True)[:15]:
    print(f"  {k:5d} {e / tot * 100:5.1f}% {s / ts * 100:5.1f}%  {data[k][isrc].strip()[:50]}")
