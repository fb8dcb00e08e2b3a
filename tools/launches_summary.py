"""Summarise an ncu --metrics launch list (csv) into profiles/ JSON.

python tools/launches_summary.py LAUNCHES.csv OUT.json "command line"
"""
import csv
import json
import statistics
import sys
from collections import defaultdict

import os
# bench.py layer launch, algorithmic bytes: Llama-3-70B (default workload); ECF8_ALGO_BYTES overrides
ALGO_PER_LAYER = int(os.environ.get("ECF8_ALGO_BYTES", "1557522886"))


def main():
    src, dst, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    rows = [r for r in csv.reader(open(src)) if len(r) > 10 and r[0] != "ID"]
    per = defaultdict(dict)
    for r in rows:
        per[(r[0], r[4])][r[12]] = float(r[14].replace(",", ""))
    by_kernel = defaultdict(list)
    for (i, name), m in per.items():
        by_kernel[name].append(m)
    total_ns = sum(m.get("gpu__time_duration.sum", 0) for ms in by_kernel.values() for m in ms)
    out = {"command": cmd, "kernels": {}}
    for name, ms in by_kernel.items():
        t = [m.get("gpu__time_duration.sum", 0) for m in ms]
        rd = [m.get("dram__bytes_read.sum", 0) for m in ms]
        wr = [m.get("dram__bytes_write.sum", 0) for m in ms]
        out["kernels"][name] = {
            "launches": len(ms), "mean_ns": statistics.mean(t), "share_of_captured_time": sum(t) / total_ns,
            "dram_read_bytes_per_launch": statistics.mean(rd), "dram_write_bytes_per_launch": statistics.mean(wr),
            "dram_bytes_per_launch": statistics.mean(rd) + statistics.mean(wr)}
    top = max(out["kernels"].items(), key=lambda kv: kv[1]["share_of_captured_time"])
    out["top_kernel"] = top[0]
    out["algorithmic_bytes_per_launch"] = ALGO_PER_LAYER
    out["achieved_gbs_cold_serialised"] = ALGO_PER_LAYER / top[1]["mean_ns"]
    out["note"] = "ncu launch times are cold-cache and serialised; compare shares, not absolutes"
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
