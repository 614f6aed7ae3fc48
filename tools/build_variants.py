"""Build tuning variants of libpot3d.so under paper_1709_01126_b200/variants/."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1709_01126_b200 import build  # noqa: E402

VARIANTS = {
    "b4m2": ["POT3D_NS_B=4", "POT3D_MINB=2"],
    "b3m2": ["POT3D_NS_B=3", "POT3D_MINB=2"],
    "b5m2": ["POT3D_NS_B=5", "POT3D_MINB=2"],
}
out = Path(build.PKG) / "variants"
out.mkdir(exist_ok=True)
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    p = build.build(defines=VARIANTS[n], out=out / f"libpot3d_{n}.so")
    print(p)
