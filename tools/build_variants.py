"""Build tuning variants of libpot3d.so under paper_1709_01126_b200/variants/."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1709_01126_b200 import build  # noqa: E402

VARIANTS = {
    "tj30": ["POT3D_TJ=30", "POT3D_MINB=1"],          # 512-thread tiles of 30 rows, 1 block/SM
    "tj22": ["POT3D_TJ=22", "POT3D_MINB=1"],          # 384 threads
    "tj30r4": ["POT3D_TJ=30", "POT3D_RPW=4", "POT3D_MINB=1"],  # 256 threads, 4 rows per lane
    "sws1": ["POT3D_SWS_MINB=1"],                     # row-scan sweeps at one CTA per SM
    "swj16m1": ["POT3D_SWJ=16", "POT3D_SWS_MINB=1"],
    "swj4": ["POT3D_SWJ=4"],
    "swj16": ["POT3D_SWJ=16"],
    "spd2": ["POT3D_SPD=2"],
    "spd3": ["POT3D_SPD=3"],
    "spd4": ["POT3D_SPD=4"],
    "pd3": [],
    "pd2": ["POT3D_SPD=2"],
    "pd4": ["POT3D_SPD=4"],
    "j4pd3": ["POT3D_SWJ=4"],
    "j16pd2": ["POT3D_SWJ=16", "POT3D_SPD=2"],
}
out = Path(build.PKG) / "variants"
out.mkdir(exist_ok=True)
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    p = build.build(defines=VARIANTS[n], out=out / f"libpot3d_{n}.so")
    print(p)
