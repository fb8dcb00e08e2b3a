"""Group SASS lines of an ncu report into basic-block-like runs (same exec
count) and print instruction and stall shares.  python tools/sass_blocks.py REP [min%]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
i, e, s = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ex = [int(r[e] or 0) for r in data]
st = [int(r[s] or 0) for r in data]
tot, stot = sum(ex), sum(st)
blocks, cur = [], None
for k, (x, r) in enumerate(zip(ex, data)):
    op = r[i].split()[0] if r[i].split() else ""
    if op.startswith("@"):
        op = r[i].split()[1]
    if cur and cur[2] == x:
        cur[1] = k
        cur[3] += st[k]
        cur[4].append(op)
    else:
        cur = [k, k, x, st[k], [op]]
        blocks.append(cur)
print(f"total warp-instr {tot}  stall samples {stot}")
for b in blocks:
    n = b[1] - b[0] + 1
    share = n * b[2] / tot * 100
    if share > thr or b[3] / stot * 100 > thr:
        ops = " ".join(sorted(set(b[4]), key=b[4].index)[:8])
        print(f"{b[0]:5d}-{b[1]:5d} n={n:3d} cnt={b[2]:9d} instr={share:5.1f}% stall={b[3] / stot * 100:5.1f}%  {ops}")
