"""Per-CUDA-source-line totals of an ncu report (instructions executed,
stall samples), from the cuda,sass source page.

python tools/ncu_lines_by_src.py REPORT [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, f, hdr, cur = {}, None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        i_ex = hdr.index("Instructions Executed")
        i_st = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0]:  # a source line row (aggregates of its SASS)
        cur = (f, int(r[0]), r[1][:80])
        try:
            agg[cur] = (int(r[i_ex] or 0), int(r[i_st] or 0))
        except (ValueError, IndexError):
            pass
tot = sum(v[0] for v in agg.values())
stot = sum(v[1] for v in agg.values())
print(f"total warp instr {tot}, stall samples {stot}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}% st{v[1] / max(stot, 1) * 100:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
