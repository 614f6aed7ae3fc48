"""Build tuning variants of libpot3d.so under paper_1709_01126_b200/variants/."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1709_01126_b200 import build  # noqa: E402

VARIANTS = {
    "strict1": ["POT3D_SWEEP_STRICT=1", "POT3D_SWEEP_PUB=1"],
    "pub1": ["POT3D_SWEEP_PUB=1"],
    "strict2": ["POT3D_SWEEP_STRICT=1"],
}
out = Path(build.PKG) / "variants"
out.mkdir(exist_ok=True)
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    p = build.build(defines=VARIANTS[n], out=out / f"libpot3d_{n}.so")
    print(p)
