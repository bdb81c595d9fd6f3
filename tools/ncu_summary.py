"""Summarise ncu reports into profiles/ (development + evidence aid).

    python tools/ncu_summary.py <report.ncu-rep> <config> [--launches launches.csv]

Writes profiles/ncu_summary.json (merged per config: duration, DRAM bytes per
launch, throughput, issue/occupancy, top stall reasons) and prints a short
markdown table.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def details(rep):
    r = ncu_csv(rep, "--page", "details")
    hdr = r[0]
    d = {}
    for row in r[1:]:
        x = dict(zip(hdr, row))
        d[x.get("Metric Name", "")] = (x.get("Metric Value", ""), x.get("Metric Unit", ""))
        d["__kernel"] = x.get("Kernel Name", "")
    return d


def raw(rep):
    r = ncu_csv(rep, "--page", "raw", "--print-units", "base")
    hdr, vals = r[0], r[2] if len(r) > 2 else r[1]
    return dict(zip(hdr, vals))


def main():
    rep, cfg = sys.argv[1], sys.argv[2]
    d = details(rep)
    rw = raw(rep)

    def num(x):
        try:
            return float(str(x).replace(",", ""))
        except Exception:
            return None
    rd = num(rw.get("dram__bytes_read.sum"))
    wr = num(rw.get("dram__bytes_write.sum"))
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v) for k, v in rw.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    stalls = dict(sorted(((k, v) for k, v in stalls.items() if v), key=lambda kv: -kv[1])[:8])
    keys = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
            "Registers Per Thread", "Achieved Active Warps Per SM", "Executed Instructions",
            "Avg. Active Threads Per Warp", "Theoretical Occupancy", "L2 Hit Rate"]
    summ = {"kernel": d.get("__kernel", "")[:120], "report": os.path.basename(rep),
            "dram_bytes_read": rd, "dram_bytes_write": wr,
            "dram_bytes_per_launch": (rd or 0) + (wr or 0) if rd is not None else None,
            "metrics": {k: " ".join(d[k]) for k in keys if k in d}, "top_stalls": stalls}
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    allv = {}
    if os.path.exists(path):
        allv = json.load(open(path))
    allv[cfg] = summ
    json.dump(allv, open(path, "w"), indent=1)
    print(f"| {cfg} | {summ['kernel'][:60]} |")
    for k, v in summ["metrics"].items():
        print(f"| {k} | {v} |")
    print(f"| DRAM bytes/launch | {summ['dram_bytes_per_launch']} |")
    print(f"| top stalls | {stalls} |")


if __name__ == "__main__":
    main()
