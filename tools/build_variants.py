"""Build kernel tuning variants of libvxb.so into build/variants/ (A/B runs
select one with VXB_LIB=...)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_01241_b200 import build as b

VARIANTS = {
    "dw4": {"VXB_DWARPS": 4},
    "dw2": {"VXB_DWARPS": 2},
    "dw3s6": {"VXB_DWARPS": 3, "VXB_STAGES": 6},
    "dw4s3e1024": {"VXB_DWARPS": 4, "VXB_STAGES": 3, "VXB_STAGE_E": 1024},
}
if __name__ == "__main__":
    out = b.ROOT / "build" / "variants"
    out.mkdir(parents=True, exist_ok=True)
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        b.build(force=True, out=out / f"libvxb_{n}.so", defines=VARIANTS[n])
        print(n)
