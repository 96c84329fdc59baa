"""Noise parity: the device Box-Muller (rng.hpp:63-67) against the reference
build's host evaluation (glibc log/cos), sample by sample."""
import ctypes as C

import numpy as np
import pytest

from paper_2308_01241_b200 import _abi
from refnet import ref_lib

pytestmark = pytest.mark.gpu


def test_ou_noise_float_samples_bit_exact():
    L, R = _abi.load_library(), ref_lib()
    rs = np.random.default_rng(1)
    n = 2_000_000
    seed = 1
    gids = rs.integers(0, 10**6, n).astype(np.uint64)
    steps = rs.integers(0, 10**5, n).astype(np.uint64)
    root = R.ref_mix_key2(seed, 1)
    base = np.array([R.ref_mix_key2(root, int(g)) for g in gids], np.uint64)
    dev = np.zeros(n, np.float64)
    assert L.vxb_debug_stream_normal(0, _abi.ptr(base), _abi.ptr(steps), n, _abi.ptr(dev)) == 0
    host = np.array([R.ref_stream_normal(int(b), int(k)) for b, k in zip(base, steps)])
    dbl_mismatch = int((dev != host).sum())
    flt_mismatch = int((dev.astype(np.float32) != host.astype(np.float32)).sum())
    print(f"double mismatches {dbl_mismatch}/{n}, float mismatches {flt_mismatch}/{n}")
    assert flt_mismatch == 0
    # the doubles may differ in the last ulp where CUDA and glibc log/cos round differently
    ulps = np.abs(dev.view(np.int64) - host.view(np.int64))
    assert ulps.max() <= 4


def test_ou_noise_float_bit_exact_1e9_samples(tmp_path):
    """1e9 (gid, step) samples — one biological second of config 2 — of the
    kernel's float xi against glibc on the host cores
    (tests/native/noise_fliprate.cu): every float sample identical."""
    import json
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    exe = tmp_path / "noise_fliprate"
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false",
                    "-Xcompiler", "-fopenmp,-ffp-contract=off",
                    "-I", str(root / "paper_2308_01241_b200" / "csrc"),
                    str(root / "tests" / "native" / "noise_fliprate.cu"), "-o", str(exe)],
                   check=True, timeout=300)
    out = subprocess.run([str(exe), "1000000", "1000", "0"], capture_output=True, text=True,
                         timeout=600, check=True).stdout
    res = json.loads(out.strip().splitlines()[-1])
    assert res["samples"] == 10**9
    assert res["float_mismatch"] == 0, res  # kernel path: fast + correctly rounded near boundaries


# (gid, step) samples where CUDA's log/cos flip the float xi against glibc
# (seed 2), found by tests/native/noise_fliprate.cu over 2e10 samples with
# the fast path alone; the kernel's stream_xi must match glibc on them.
FAST_PATH_FLIPS = [(1274108, 1240), (3587472, 477), (3964552, 1179), (4635374, 1866),
                   (5995597, 1274), (6881677, 1518), (7567786, 1090), (8835931, 68),
                   (9739371, 858)]


def test_ou_noise_near_boundary_samples_match_glibc():
    L, R = _abi.load_library(), ref_lib()
    root = R.ref_mix_key2(2, 1)
    base = np.array([R.ref_mix_key2(root, g) for g, _ in FAST_PATH_FLIPS], np.uint64)
    steps = np.array([t for _, t in FAST_PATH_FLIPS], np.uint64)
    n = len(base)
    fast = np.zeros(n, np.float64)
    xi = np.zeros(n, np.float32)
    assert L.vxb_debug_stream_normal(0, _abi.ptr(base), _abi.ptr(steps), n, _abi.ptr(fast)) == 0
    assert L.vxb_debug_stream_xi(0, _abi.ptr(base), _abi.ptr(steps), n, _abi.ptr(xi)) == 0
    host = np.array([R.ref_stream_normal(int(b), int(k)) for b, k in zip(base, steps)]).astype(np.float32)
    assert (fast.astype(np.float32) != host).all()  # the fast path really flips here
    assert np.array_equal(xi, host)


def test_correctly_rounded_normal_agrees_with_glibc(tmp_path):
    """The double-double stream_normal_cr (used near rounding boundaries for
    the OU noise and the Q16 synapse weights) is correctly rounded: it
    differs from glibc only where glibc itself is not (log ~0.08 %, cos
    ~0.13 % of inputs, checked against mpmath), against ~15 % for CUDA's
    fast log/cos (tests/native/normal_cr_check.cu, 2e7 samples)."""
    import json
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    exe = tmp_path / "normal_cr_check"
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false",
                    "-Xcompiler", "-fopenmp,-ffp-contract=off",
                    "-I", str(root / "paper_2308_01241_b200" / "csrc"),
                    str(root / "tests" / "native" / "normal_cr_check.cu"), "-o", str(exe)],
                   check=True, timeout=300)
    res = json.loads(subprocess.run([str(exe), "20000000"], capture_output=True, text=True,
                                    timeout=600, check=True).stdout.strip().splitlines()[-1])
    assert res["cr_double_mismatch"] < 0.004 * res["samples"], res
    assert res["fast_double_mismatch"] > 0.1 * res["samples"], res
