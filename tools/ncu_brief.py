"""Headline metrics of an ncu report (time, issue, pipes, stalls, DRAM, smem).

python tools/ncu_brief.py REPORT
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.sum.per_cycle_active",
        "sm__inst_executed.sum.per_cycle_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    print("kernel:", r[h.index("Kernel Name")][:100])
    for k in keys:
        if k in h:
            print(f"  {k:70s} {r[h.index(k)]:>16s} {u[h.index(k)]}")
    st = [(n, float(r[i] or 0)) for i, n in enumerate(h)
          if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
    st.sort(key=lambda x: -x[1])
    print("  stalls/issue:", ", ".join(f"{n[35:-29]} {v:.2f}" for n, v in st[:9]))
