"""Build tuning variants of libpot3d.so under paper_1709_01126_b200/variants/."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1709_01126_b200 import build  # noqa: E402

VARIANTS = {
    "base": [],
    "r1m2": ["POT3D_RPW=1", "POT3D_MINB=2"],
    "r1m1": ["POT3D_RPW=1", "POT3D_MINB=1"],
}
out = Path(build.PKG) / "variants"
out.mkdir(exist_ok=True)
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    p = build.build(defines=VARIANTS[n], out=out / f"libpot3d_{n}.so")
    print(p)
