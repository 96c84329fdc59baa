"""Build the CUDA engine (libvxb.so) in-tree for sm_100a.

    python -m paper_2308_01241_b200.build [-v]

nvcc cross-compiles without a GPU.  The shared object is written next to this
file so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libvxb.so"
MARKER = b"VXB_SRC_HASH="

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "--fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O3,-fopenmp",
    "-shared", "-lcudart", "-lgomp",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and Path(c).exists():
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return [CSRC / "vxb_engine.cu"]


def deps():
    return sources() + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "vxb.h"]


def source_hash(defines: dict | None = None) -> str:
    """SHA-256 (first 32 hex digits) over every source, header and compiler
    flag of the build.  It is compiled into the library (vxb_build_hash) and
    decides freshness: a copy that preserves mtimes cannot hide a stale .so."""
    h = hashlib.sha256()
    for p in sorted(deps()):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join([*ARCH, *NVCC_FLAGS]).encode())
    h.update(repr(sorted((defines or {}).items())).encode())
    return h.hexdigest()[:32]


def built_hash(path: Path = OUT) -> str | None:
    """The source hash embedded in a built library (marker string), or None."""
    try:
        data = path.read_bytes()
    except OSError:
        return None
    k = data.find(MARKER)
    if k < 0:
        return None
    return data[k + len(MARKER):k + len(MARKER) + 32].decode("ascii", "replace")


def up_to_date() -> bool:
    return built_hash(OUT) == source_hash()


def build(verbose: bool = False, force: bool = False, out: Path = OUT,
          defines: dict | None = None) -> Path:
    """Compile libvxb.so; `defines` (-D) select kernel tuning variants."""
    if not force and out == OUT and up_to_date():
        return OUT
    dflags = [f"-D{k}={v}" for k, v in (defines or {}).items()]
    dflags.append(f"-DVXB_SRC_HASH=\"{source_hash(defines)}\"")
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *dflags, f"-I{ROOT / 'include'}", f"-I{CSRC}",
           *(str(s) for s in sources()), "-o", str(out) + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(str(out) + ".tmp", out)
    return out


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force=True)
    print(OUT)
