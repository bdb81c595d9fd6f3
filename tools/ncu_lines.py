"""Per-source-line totals of an ncu capture: joins `ncu --page source --csv
--print-source sass` (per-instruction counters) with the line table of
`nvdisasm -g` on the kernel's cubin.

    python tools/ncu_lines.py sass.csv all.dis <mangled kernel name> [file filter]
"""
import csv
import re
import sys
from collections import defaultdict

sass_csv, dis, kern = sys.argv[1:4]
filt = sys.argv[4] if len(sys.argv) > 4 else ""
# line table: address -> (file, line) inside the kernel's text section
addr2line = {}
cur = None
insec = False
for ln in open(dis, errors="replace"):
    if ln.startswith("\t.section") or ln.startswith(".section"):
        insec = (".text." + kern) in ln
        continue
    if not insec:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+\S", ln)
    if m and cur:
        addr2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ia, ie, ismp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("# Samples")
base = None
tot = defaultdict(lambda: [0, 0])
total = 0
for r in rows[2:]:
    if len(r) <= ie:
        continue
    a = int(r[ia], 16) if r[ia].startswith("0x") else int(r[ia])
    if base is None:
        base = a
    key = addr2line.get(a - base, ("?", 0))
    n = int(r[ie] or 0)
    tot[key][0] += n
    tot[key][1] += int(r[ismp] or 0)
    total += n
print("total instructions", total)
src = {}
for (f, l), (n, s) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:60]:
    if filt and filt not in f:
        pass
    if f not in src:
        try:
            src[f] = open("/root/repo/paper_2506_04165_b200/csrc/" + f).read().split("\n")
        except OSError:
            src[f] = []
    text = src[f][l - 1].strip()[:90] if 0 < l <= len(src[f]) else ""
    print(f"{n:>9} {100.0 * n / total:5.1f}% smp {s:>6}  {f}:{l}  {text}")
