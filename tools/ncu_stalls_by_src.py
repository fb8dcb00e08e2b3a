"""Per-CUDA-line stall reasons of an ncu report (cuda,sass source page).

python tools/ncu_stalls_by_src.py REPORT [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, f, hdr = {}, None, None
reasons = []
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
        reasons = [(i, n) for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
        i_all = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0]:
        try:
            key = (f, int(r[0]), r[1][:60])
            agg[key] = (int(r[i_all] or 0), {n: int(r[i] or 0) for i, n in reasons})
        except (ValueError, IndexError):
            pass
tot = sum(v[0] for v in agg.values())
by_reason = {}
for k, (n, d) in agg.items():
    for rn, c in d.items():
        by_reason[rn] = by_reason.get(rn, 0) + c
print("total samples", tot, " by reason:", ", ".join(f"{k[6:]} {v * 100 / tot:.1f}%" for k, v in
                                                    sorted(by_reason.items(), key=lambda x: -x[1])[:8]))
for k, (n, d) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    rs = ", ".join(f"{rn[6:]} {c}" for rn, c in sorted(d.items(), key=lambda x: -x[1])[:3] if c)
    print(f"{n * 100 / tot:5.1f}%  {k[0]}:{k[1]}  [{rs}]  {k[2]}")
