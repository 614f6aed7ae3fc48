"""Count SASS instructions inside the loop(s) containing BAR.SYNC of each kernel.
   python tools/sass_loop.py file.o|.so [kernel-substring]"""
import re
import subprocess
import sys
from collections import Counter

obj = sys.argv[1]
filt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if filt not in name:
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, s) in enumerate(ins):
        if "BRA" not in s:
            continue
        t = re.search(r"0x([0-9a-f]+)", s)
        if t:
            tgt = int(t.group(1), 16)
            if tgt < a and tgt in addr:
                body = ins[addr[tgt]:i + 1]
                if any("BAR.SYNC" in b for _, b in body):
                    loops.append((addr[tgt], i, body))
    print(f"== {name[:60]}: {len(ins)} instructions")
    for lo, hi, body in loops:
        c = Counter(re.sub(r"^@!?U?P\w+\s+", "", b).split()[0].split(".")[0] for _, b in body)
        print(f"   loop [{lo},{hi}] {len(body)} instr: " + ", ".join(f"{k}:{v}" for k, v in c.most_common(16)))
