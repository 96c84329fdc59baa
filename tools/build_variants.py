"""Build kernel tuning variants of libvxb.so into build/variants/ (A/B runs
select one with VXB_LIB=...)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_01241_b200 import build as b

VARIANTS = {
    "dw3s4e1024": {"VXB_DWARPS": 3, "VXB_STAGES": 4, "VXB_STAGE_E": 1024},
    "dw3s6e768": {"VXB_DWARPS": 3, "VXB_STAGES": 6, "VXB_STAGE_E": 768},
    "dw3s3e1536": {"VXB_DWARPS": 3, "VXB_STAGES": 3, "VXB_STAGE_E": 1536},
    "dw3s2e768": {"VXB_DWARPS": 3, "VXB_STAGES": 2, "VXB_STAGE_E": 768},
}
if __name__ == "__main__":
    out = b.ROOT / "build" / "variants"
    out.mkdir(parents=True, exist_ok=True)
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        b.build(force=True, out=out / f"libvxb_{n}.so", defines=VARIANTS[n])
        print(n)
