"""Build kernel tuning variants of libvxb.so into build/variants/ (A/B runs
select one with VXB_LIB=...)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_01241_b200 import build as b

VARIANTS = {
    # tile path (vxb_tile.cuh)
    "tt768": {"VXB_TILE_THREADS": 768},    # 24 warps at 80 registers
    "tt640": {"VXB_TILE_THREADS": 640},    # 20 warps at 96 registers
    "tt896": {"VXB_TILE_THREADS": 896},    # 28 warps at 72 registers
    "tt960": {"VXB_TILE_THREADS": 960},    # 30 warps at 68 registers
    "tt768u8": {"VXB_TILE_THREADS": 768, "VXB_TILE_UNROLL": 8},
    "u8": {"VXB_TILE_UNROLL": 8},
    "u2": {"VXB_TILE_UNROLL": 2},
    "u5": {"VXB_TILE_UNROLL": 5},
    "u6": {"VXB_TILE_UNROLL": 6},
    "l1pf": {"VXB_TILE_L1PF": 1},
    "scan1": {"VXB_TILE_SCANW": 1},   # one warp scans the peers' batches
    "scan4": {"VXB_TILE_SCANW": 4},
    "spin2": {"VXB_TILE_SPIN0": 200, "VXB_TILE_SPIN1": 500},   # longer sleeps while waiting for the queues
    "spin3": {"VXB_TILE_SPIN0": 500, "VXB_TILE_SPIN1": 1000},
    "nopf": {"VXB_TILE_L1PF": 0},          # no L1 prefetch of the chunk after next
    "bw4": {"VXB_TILE_BWARPS": 4},
    "bw6": {"VXB_TILE_BWARPS": 6},
    "bw8": {"VXB_TILE_BWARPS": 8},
    "nofuse": {"VXB_TILE_FUSE_NOISE": 0},
    "pf48": {"VXB_TILE_PREFETCH": 48},     # L2 prefetch distance in queue items
    "pf64": {"VXB_TILE_PREFETCH": 64},
    "pf96": {"VXB_TILE_PREFETCH": 96},
    "pf12": {"VXB_TILE_PREFETCH": 12},  # the OU step as a separate pass after the update
    # l2_atomic path (vxb_kernels.cuh)
    "m2": {"VXB_MINB": 2},           # register cap lifted (2 CTAs/SM)
    "d3": {"VXB_DEPTH3": 1},         # update state two chunks ahead in registers
    # diagnostic, not parity-preserving: cost of the OU noise
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
