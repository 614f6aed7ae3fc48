"""Hottest SASS lines of a kernel in an ncu report by a stall column:
   python tools/ncu_hot.py rep.ncu-rep kernel_regex [column] [n]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
col = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
n = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ci = hdr.index(col)
si = hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[si] or 0) for r in body)
body.sort(key=lambda r: -int(r[ci] or 0))
print(f"total samples {tot}; top by {col}")
idx = {r[0]: i for i, r in enumerate(rows[2:])}
for r in body[:n]:
    print(f"{int(r[ci] or 0):7d} {int(r[si] or 0):7d}  {r[0][-5:]}  {r[1].strip()[:90]}")
