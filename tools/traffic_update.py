"""profiles/traffic.json from an ncu --set full report: per kernel (base name), the
mean dram__bytes_read.sum + dram__bytes_write.sum per launch.
   python tools/traffic_update.py report.ncu-rep config"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

rep, config = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
iname, ird, iwr = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
acc = defaultdict(list)
for r in rows[2:]:
    name = re.sub(r"^(void )?(pot3d::)?", "", r[iname]).split("(")[0].split("<")[0]
    b = float(r[ird]) * scale[units[ird]] + float(r[iwr]) * scale[units[iwr]]
    acc[name].append(b)
p = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
d = json.loads(p.read_text()) if p.exists() else {}
d[config] = {k: int(sum(v) / len(v)) for k, v in acc.items()}
d[config]["_note"] = (f"ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch, mean over "
                      f"{sum(len(v) for v in acc.values())} launches ({Path(rep).name})")
p.write_text(json.dumps(d, indent=1) + "\n")
print(json.dumps(d[config], indent=1))
