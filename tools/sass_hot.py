"""Hot SASS lines of an ncu report (instructions executed + stall samples).

python tools/sass_hot.py REPORT [min_pct]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
i_st = hdr.index("Warp Stall Sampling (All Samples)")
ex = [int(r[i_ex] or 0) for r in data]
st = [int(r[i_st] or 0) for r in data]
tot, stot = sum(ex), sum(st)
print(f"total warp instr {tot}, stall samples {stot}, sass lines {len(data)}")
for k, r in enumerate(data):
    if ex[k] > tot * thr / 100 or st[k] > stot * 0.01:
        print(f"{k:4d} {ex[k] / tot * 100:5.2f}% st{st[k] / stot * 100:5.1f}% {r[i_src][:90]}")
