"""Hottest SASS instructions of one kernel in an ncu report (stall samples), and
the instruction mix weighted by executed count.
   python tools/ncu_sass_hot.py rep.ncu-rep kernel-regex [top]"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = raw.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
iS, iE, iT, iD = (hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"),
                  hdr.index("Thread Instructions Executed"), hdr.index("Divergent Branches"))
data = []
for r in rows[1:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        break
    data.append((r[0], r[1].strip(), int(r[iS] or 0), int(r[iE] or 0), int(r[iT] or 0), int(r[iD] or 0)))
tot_s = sum(d[2] for d in data) or 1
tot_e = sum(d[3] for d in data) or 1
print(f"{len(data)} SASS lines, {tot_e} warp instructions, {tot_s} stall samples")
mix = Counter()
for d in data:
    op = re.sub(r"^@!?U?P\w+\s+", "", d[1]).split()[0].split(".")[0]
    mix[op] += d[3]
print("mix:", ", ".join(f"{k} {100 * v / tot_e:.1f}%" for k, v in mix.most_common(24)))
print("divergent branches:", sum(d[5] for d in data))
for d in sorted(data, key=lambda d: -d[2])[:top]:
    print(f"{100 * d[2] / tot_s:5.1f}% {d[3]:>10} {d[4] / max(d[3], 1):5.1f}thr  {d[1][:90]}")

if len(sys.argv) > 4:  # context around the hottest lines
    hot = sorted(range(len(data)), key=lambda i: -data[i][2])[: int(sys.argv[4])]
    for h in hot:
        print("----")
        for i in range(max(0, h - 6), min(len(data), h + 3)):
            d = data[i]
            print(f"{'>>' if i == h else '  '} {100 * d[2] / tot_s:5.1f}% {d[3]:>10}  {d[1][:100]}")
