"""CPU tests: the C restatement (oracle/voxsim_oracle.c) pinned against the
reference's known-answer tests, the golden fixtures generated from the
reference build (tests/golden/make_golden.py), and the reference engine itself
on identical tables."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2308_01241_b200.engine import ConfigError, ForcedSpike, Injection, SimError, SimOptions
from refnet import OracleSim, RefNet, RefSim, make_config, oracle_lib, raster_set, ref_lib

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def O():
    return oracle_lib()


# test_rng.cpp:13-21
def test_stream_word_frozen(O):
    assert O.vxo_stream_word(0x0, 0) == 0xe220a8397b1dcdaf
    assert O.vxo_stream_word(0x0, 1) == 0x6e789e6aa1b965f4
    assert O.vxo_stream_word(0x1, 0) == 0x910a2dec89025cc1
    assert O.vxo_stream_word(0xdeadbeef, 7) == 0xb30a4ccf430b1b5a
    assert O.vxo_stream_word(123456789, 1000000) == 0xb2957a36c8d58985


# test_rng.cpp:23-35
def test_stream_u01_frozen(O):
    for k, want in enumerate([0.7415648787718233, 0.1599103928769201, 0.27860113025513866,
                              0.34419071652363753]):
        assert abs(O.vxo_stream_u01(42, k) - want) <= 1e-15 * want
    u = [O.vxo_stream_u01(7, k) for k in range(1000)]
    assert min(u) >= 0.0 and max(u) < 1.0


def test_rng_golden_fixture(O):
    g = json.loads((GOLD / "rng.json").read_text())
    for b, k, w in g["stream_word"]:
        assert O.vxo_stream_word(b, k) == w
    for b, k, h in g["stream_u01"]:
        assert O.vxo_stream_u01(b, k) == float.fromhex(h)
    for a, b, w in g["mix_key"]:
        assert O.vxo_mix_key(a, b) == w
    for b, k, n, w in g["stream_below"]:
        assert O.vxo_stream_below(b, k, n) == w
    for b, k, h in g["stream_normal"]:
        assert O.vxo_stream_normal(b, k) == float.fromhex(h)
    for w, q in g["quantize"]:
        assert O.vxo_quantize_weight(w) == q


def test_ou_noise_golden_fixture(O):
    z = np.load(GOLD / "xi.npz")
    for a, s in enumerate(z["seeds"]):
        for b in range(0, len(z["gids"]), 37):
            for c in range(0, len(z["steps"]), 11):
                got = O.vxo_ou_xi(int(s), int(z["gids"][b]), int(z["steps"][c]))
                assert np.float32(got) == z["xi"][a, b, c]


# test_rng.cpp:123-139
def test_stream_normal_moments(O):
    base = O.vxo_mix_key(O.vxo_mix_key(5, 1), 17)
    z = np.array([O.vxo_stream_normal(base, k) for k in range(200000)])
    assert abs(z.mean()) < 0.01
    assert abs(z.var() - 1.0) < 0.01


# test_model.cpp:35-223 exact kernel values
def test_model_kernels_exact(O):
    assert O.vxo_gating_kernel(1.5, 1.0, 4.0, 0.5, 1.25) == 1.75
    g = (C.c_float * 4)(2.0, 0.0, 0.0, 0.0)
    j = (C.c_float * 4)(1.0, 0.0, 0.0, 0.0)
    e = (C.c_float * 4)(0.0, 0.0, -70.0, -70.0)
    assert O.vxo_current_kernel(-70.0, j, g, e) == 140.0
    g = (C.c_float * 4)(0.0, 0.0, 4.0, 0.0)
    j = (C.c_float * 4)(0.0, 0.0, 1.0, 0.0)
    assert O.vxo_current_kernel(-60.0, j, g, e) == -40.0
    assert O.vxo_membrane_kernel(-65.0, 1.0 / 250.0, 25.0, -65.0, 1000.0, 625.0) == -58.5
    assert O.vxo_ou_kernel(0.0, 1.0, 250.0, 0.0, 10.0, 0.0) == 25.0
    assert O.vxo_quantize_weight(0.0) == 0
    assert O.vxo_quantize_weight(-3.5) == 0
    assert O.vxo_quantize_weight(1.0) == 65536
    assert O.vxo_dequantize_weight(65536) == 1.0
    assert O.vxo_dequantize_weight(32768) == 0.5


def test_kernels_match_reference_build(O):
    R = ref_lib()
    rs = np.random.default_rng(0)
    for _ in range(2000):
        a = rs.uniform(-80, 10, 6).astype(np.float32)
        assert O.vxo_membrane_kernel(*map(float, a)) == R.ref_membrane_kernel(*map(float, a))
        b = np.abs(rs.normal(1, 2, 5)).astype(np.float32) + np.float32(1e-3)
        assert O.vxo_gating_kernel(*map(float, b)) == R.ref_gating_kernel(*map(float, b))
        c = rs.normal(0, 100, 6).astype(np.float32)
        c[4] = abs(c[4]) + 1
        c[1] = abs(c[1]) / 100 + np.float32(0.01)
        assert O.vxo_ou_kernel(*map(float, c)) == R.ref_ou_kernel(*map(float, c))
        q = int(rs.integers(-2**40, 2**40))
        assert O.vxo_dequantize_weight(q) == R.ref_dequantize_weight(q)
        w = float(rs.normal(1, 3))
        assert O.vxo_quantize_weight(w) == R.ref_quantize_weight(w)
        key = int(rs.integers(0, 2**63))
        k = int(rs.integers(0, 2**40))
        assert O.vxo_stream_normal(key, k) == R.ref_stream_normal(key, k)


def _golden_run(name):
    z = np.load(GOLD / f"{name}.npz")
    cfg = json.loads(str(z["cfg"]))
    return z, cfg


@pytest.mark.parametrize("name,opt", [
    ("six_neurons", SimOptions(steps=150, probe_gids=list(range(6)))),
    ("ring3_w3", SimOptions(steps=120, probe_gids=[7, 179])),
    ("hot_forced", SimOptions(steps=30, forced_spikes=[ForcedSpike(4, 2)], probe_gids=[2])),
])
def test_oracle_matches_golden_runs(name, opt):
    z, cfg = _golden_run(name)
    net = RefNet(cfg, even_workers=int(z["even"]))
    r = OracleSim(net.tables, opt).advance(opt.steps)
    keys = np.array(raster_set(r.raster), np.uint64).reshape(-1, 2)
    assert np.array_equal(keys, z["raster"])
    assert np.array_equal(r.rates, z["rates"])
    assert np.array_equal(r.probe_v, z["probe_v"])
    assert np.array_equal(r.probe_i, z["probe_i"])
    assert list(r.flops.values()) == z["flops"].tolist()


@pytest.mark.parametrize("workers,cfg", [
    (1, make_config(seed=9, voxels=1, npv=300, k_in=30, ou_mean=300.0)),
    (2, make_config(seed=4, voxels=4, npv=150, k_in=20, rho=0.25)),
    (3, make_config(seed=44, voxels=3, npv=50, k_in=6, rho=0.5)),
])
def test_oracle_matches_reference_engine(workers, cfg):
    net = RefNet(cfg, even_workers=workers)
    inj = [Injection(5, 40, 0, 300.0), Injection(20, 60, 0, -120.0)]
    opt = SimOptions(steps=80, probe_gids=[0, 13, 149], injections=inj,
                     forced_spikes=[ForcedSpike(3, 1), ForcedSpike(9, 13)])
    rs = RefSim(net, opt)
    ref = rs.advance(50)
    ref2 = rs.advance(30)
    orc = OracleSim(net.tables, opt)
    o = orc.advance(50)
    o2 = orc.advance(30)
    for a, b in ((ref, o), (ref2, o2)):
        assert a.total_spikes == b.total_spikes
        assert raster_set(a.raster) == raster_set(b.raster)
        assert np.array_equal(a.rates, b.rates)
        assert np.array_equal(a.probe_v, b.probe_v)
        assert np.array_equal(a.probe_i, b.probe_i)
        assert a.flops == b.flops
    for w in range(workers):
        assert np.array_equal(rs.membrane_snapshot(w), orc.membrane_snapshot(w))


def test_survey_golden_counts():
    counts = json.loads((GOLD / "counts.json").read_text())
    assert counts["config1_dt0.1_10000"] == 33078
    assert counts["config1_dt1_1000"] == 35702
    net = RefNet(make_config(seed=1, voxels=1, npv=10000, k_in=100, dt_ms=1.0, steps=1000))
    r = OracleSim(net.tables, SimOptions(steps=300, record_raster=False)).advance(300)
    ref = RefSim(net, SimOptions(steps=300, record_raster=False)).advance(300)
    assert r.total_spikes == ref.total_spikes


def test_oracle_error_behaviour():
    net = RefNet(make_config(seed=1, voxels=3, npv=20, k_in=2, ou_mean=0.0, ou_sigma=0.0))
    with pytest.raises(ConfigError):
        OracleSim(net.tables, SimOptions(dt_ms=0.0))
    with pytest.raises(ConfigError):
        OracleSim(net.tables, SimOptions(injections=[Injection(0, 5, 99, 1.0)]))
    with pytest.raises(SimError):
        OracleSim(net.tables, SimOptions(probe_gids=[10**6]))
    o = OracleSim(net.tables, SimOptions(injections=[Injection(0, 10, 0, float("inf"))]))
    with pytest.raises(SimError, match="diverged"):
        o.advance(5)
