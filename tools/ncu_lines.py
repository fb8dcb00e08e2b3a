"""Per-CUDA-source-line instruction and stall shares of an ncu report
(ncu --page source --print-source=cuda,sass), aggregated over all files.

python tools/ncu_lines.py REPORT [min_pct]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
fname = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue  # cuda rows only (sass rows carry an Address)
    d = dict(zip(hdr[4:], r[4:]))
    num = lambda k: int(d.get(k)) if (d.get(k) or "").isdigit() else 0
    ex = num("Instructions Executed")
    th = num("Thread Instructions Executed")
    st = num("Warp Stall Sampling (All Samples)")
    if ex or st:
        agg[(fname, int(r[0]))] = (ex, th, st, r[1].strip(), num("stall_long_sb"), num("stall_short_sb"),
                                   num("stall_wait"))
tot = sum(v[0] for v in agg.values()) or 1
stot = sum(v[2] for v in agg.values()) or 1
print(f"total warp instr {tot}, stall samples {stot}")
print(" instr%  stall% (long short wait)  thr/warp  line")
for (f, ln), (ex, th, st, src, sl, ss, sw) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if ex / tot * 100 >= thr or st / stot * 100 >= thr:
        print(f"{ex / tot * 100:5.1f}% {st / stot * 100:5.1f}% ({sl / stot * 100:4.1f} {ss / stot * 100:4.1f} "
              f"{sw / stot * 100:4.1f}) {th / max(ex, 1):5.1f} {f}:{ln} {src[:70]}")
