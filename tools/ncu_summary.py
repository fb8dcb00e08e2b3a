"""Summarise an ncu report: key metrics + per-region SASS instruction shares.

python tools/ncu_summary.py REPORT.ncu-rep [--sass]
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Executed Instructions", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Eligible Warps Per Scheduler", "No Eligible", "Dynamic Shared Memory Per Block", "Branch Efficiency",
        "Grid Size", "SM Frequency", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        res[d.get("Metric Name")] = (d.get("Metric Value"), d.get("Metric Unit"))
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {n: (vals[hdr.index(n)], units[hdr.index(n)]) for n in names if n in hdr}


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, vals = rows[0], rows[2]
    res = []
    for h, v in zip(hdr, vals):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                res.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    return sorted(res, reverse=True)[:10]


if __name__ == "__main__":
    rep = sys.argv[1]
    d = details(rep)
    for k in KEYS:
        if k in d:
            print(f"{k:40s} {d[k][0]} {d[k][1]}")
    for k, v in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                          "sm__inst_executed.sum", "smsp__inst_executed.sum"]).items():
        print(f"{k:40s} {v[0]} {v[1]}")
    print("top stall reasons (warps per issue):")
    for v, n in stalls(rep):
        print(f"   {n:30s} {v:.2f}")
