"""Build kernel tuning variants of libvxb.so into build/variants/ (A/B runs
select one with VXB_LIB=...)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_01241_b200 import build as b

VARIANTS = {
    "dw4": {"VXB_DWARPS": 4},
    "dw5": {"VXB_DWARPS": 5},
    "dw4s6e512": {"VXB_DWARPS": 4, "VXB_STAGES": 6, "VXB_STAGE_E": 512},
    "dw4s8e384": {"VXB_DWARPS": 4, "VXB_STAGES": 8, "VXB_STAGE_E": 384},
    "t384dw6": {"VXB_THREADS": 384, "VXB_MINB": 2, "VXB_DWARPS": 6},
}
if __name__ == "__main__":
    out = b.ROOT / "build" / "variants"
    out.mkdir(parents=True, exist_ok=True)
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        b.build(force=True, out=out / f"libvxb_{n}.so", defines=VARIANTS[n])
        print(n)
