"""Build tuning variants of libpot3d.so under paper_1709_01126_b200/variants/."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1709_01126_b200 import build  # noqa: E402

VARIANTS = {
    "sd4m3": ["POT3D_SWEEP_D=4", "POT3D_SWEEP_MINB=3"],
    "sd4m4": ["POT3D_SWEEP_D=4", "POT3D_SWEEP_MINB=4"],
    "sd2m4": ["POT3D_SWEEP_D=2", "POT3D_SWEEP_MINB=4"],
    "sd8m2": ["POT3D_SWEEP_D=8", "POT3D_SWEEP_MINB=2"],
}
out = Path(build.PKG) / "variants"
out.mkdir(exist_ok=True)
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    p = build.build(defines=VARIANTS[n], out=out / f"libpot3d_{n}.so")
    print(p)
