"""Build kernel tuning variants of libvxb.so into build/variants/ (A/B runs
select one with VXB_LIB=...)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_01241_b200 import build as b

VARIANTS = {
    "m4": {"VXB_MINB": 4},
    "t384m2": {"VXB_THREADS": 384, "VXB_MINB": 2},
    "t384m2dw4": {"VXB_THREADS": 384, "VXB_MINB": 2, "VXB_DWARPS": 4},
    "t512m2dw4": {"VXB_THREADS": 512, "VXB_MINB": 2, "VXB_DWARPS": 4},
    "t320m3": {"VXB_THREADS": 320, "VXB_MINB": 3},
    "polsf": {"VXB_POL_STREAM": 0},  # synapse stream evict_first
    "polkn": {"VXB_POL_KEEP": 1},    # pending evict_normal
    "pf1": {"VXB_PREFETCH": 1},      # L2 prefetch of the update state two chunks ahead
    "dw4": {"VXB_DWARPS": 4},        # 1 producer + 3 consumer warps per CTA
    "dw2": {"VXB_DWARPS": 2},        # 1 producer + 1 consumer
    "s6": {"VXB_STAGES": 6},         # deeper bulk-copy ring
    "s3": {"VXB_STAGES": 3},
    "e1024": {"VXB_STAGE_E": 1024},  # larger stages
    "e512": {"VXB_STAGE_E": 512},
    "m2": {"VXB_MINB": 2},           # register cap lifted (2 CTAs/SM)
    "d3": {"VXB_DEPTH3": 1},         # update state two chunks ahead in registers
    "d3m2": {"VXB_DEPTH3": 1, "VXB_MINB": 2},  # same, register cap lifted (2 CTAs/SM)
    # diagnostic, not parity-preserving: cost of the OU noise in the update
    "xifast": {"VXB_XI_FAST_ONLY": 1},  # fp64 Box-Muller without the correct-rounding check
    "xizero": {"VXB_XI_ZERO": 1},       # no noise at all
}
if __name__ == "__main__":
    out = b.ROOT / "build" / "variants"
    out.mkdir(parents=True, exist_ok=True)
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        b.build(force=True, out=out / f"libvxb_{n}.so", defines=VARIANTS[n])
        print(n)
