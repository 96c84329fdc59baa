"""GPU parity of the BOLD-proxy readout (vxb_hemo.cuh) against the reference's
hemodynamics (hemo.cpp via oracle/_ref) and window_bold drive (assim.cpp:51-71).

The Balloon-Windkessel step is the reference's arithmetic operation for
operation in IEEE double; only pow() differs (CUDA's vs glibc's, each within
an ulp), so states and BOLD are compared at 1e-12 relative (BOLD at 1e-12 of
its scale plus 1e-15 absolute), the rest fixed point exactly."""
import numpy as np
import pytest

from paper_2308_01241_b200.engine import (ConfigError, HemoParams, SimError, SimInstance,
                                          SimOptions, bold_from_drive, hemo_rest)
from refnet import RefNet, RefSim, make_config, ref_bold_from_drive, ref_window_bold

pytestmark = pytest.mark.gpu


def close(a, b, rel=1e-12):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(1e-300, float(np.max(np.abs(b))) if b.size else 1.0)
    return np.max(np.abs(a - b)) <= rel * scale + 1e-15 if a.size else True


# test_hemo.cpp:35-45
def test_rest_is_an_exact_fixed_point():
    st = hemo_rest(1)
    b = bold_from_drive(np.zeros(5000), 0.001, 1, state=st)
    assert np.all(b == 0.0)
    assert (st["s"][0], st["f"][0], st["v"][0], st["q"][0]) == (0.0, 1.0, 1.0, 1.0)


# test_hemo.cpp:47-61
def test_one_euler_step_matches_hand_computed_reference():
    st = hemo_rest(1)
    st["s"], st["f"], st["v"], st["q"] = 0.1, 1.2, 1.1, 0.9
    b = bold_from_drive([0.5], 0.01, 1, state=st)
    assert st["s"][0] == pytest.approx(0.10353000000000001, rel=1e-14)
    assert st["f"][0] == pytest.approx(1.201, rel=1e-14)
    assert st["v"][0] == pytest.approx(1.0985004891109096, rel=1e-12)
    assert st["q"][0] == pytest.approx(0.8992950357636457, rel=1e-12)
    assert b[0] == pytest.approx(0.01110167448431187, rel=1e-10)


# test_hemo.cpp:63-89
def test_boxcar_delayed_peak_undershoot_recovery():
    z = np.zeros(30000)
    z[:1000] = 1.0
    b = bold_from_drive(z, 0.001, 1)
    t_peak, t_dip = int(np.argmax(b)), int(np.argmin(b))
    assert b.max() > 0.02 and 2500 < t_peak < 4500
    assert b.min() < -0.002 and t_dip > t_peak
    assert abs(b[-1]) < 1e-4 and abs(b[99]) < 1e-3
    assert close(b, ref_bold_from_drive(HemoParams(), z, 0.001, 1))


# test_hemo.cpp:91-106
def test_sustained_drive_saturates():
    b = bold_from_drive(np.ones(20000), 0.001, 1)
    assert b.max() == pytest.approx(0.0481, rel=0.02)
    assert 0.0 < b[-1] < b.max()


# test_hemo.cpp:108-134
def test_sampling_and_state_carry_over():
    z = np.full(1000, 0.7)
    sampled = bold_from_drive(z, 0.001, 100)
    dense = bold_from_drive(z, 0.001, 1)
    assert sampled.size == 10 and sampled[0] == dense[99] and sampled[9] == dense[999]
    st = hemo_rest(1)
    a = bold_from_drive(z[:500], 0.001, 100, state=st)
    b = bold_from_drive(z[500:], 0.001, 100, state=st)
    assert np.array_equal(np.concatenate([a, b]), sampled)
    with pytest.raises(ConfigError):
        bold_from_drive(z, 0.001, 0)


# test_hemo.cpp:136-141
def test_state_divergence_raises_sim_error():
    st = hemo_rest(1)
    st["s"] = np.inf
    with pytest.raises(SimError, match="hemodynamic state diverged"):
        bold_from_drive([0.0], 0.001, 1, state=st)


def test_random_drives_match_reference():
    rng = np.random.default_rng(11)
    z = rng.gamma(2.0, 0.6, size=(64, 4000))
    st = hemo_rest(64)
    b = bold_from_drive(z, 0.001, 40, state=st)
    for i in range(64):
        sr = np.array([0.0, 1.0, 1.0, 1.0])
        rb = ref_bold_from_drive(HemoParams(), z[i], 0.001, 40, sr)
        assert close(b[i], rb)
        assert close([st["s"][i], st["f"][i], st["v"][i], st["q"][i]], sr)


# window_bold on the engine's own rate series, carried over two advances
def test_engine_bold_readout_matches_reference_window_bold():
    net = RefNet(make_config(seed=7, voxels=3, npv=200, k_in=20, rho=0.3, ou_mean=400.0,
                             ou_sigma=150.0), even_workers=2)
    opt = SimOptions(steps=400, dt_ms=1.0)
    units = net.tables.units
    vox_n = np.zeros(net.tables.n_voxels, np.uint64)
    np.add.at(vox_n, units["voxel"].astype(np.int64), units["neurons"].astype(np.uint64))
    with SimInstance(net.tables, opt) as sim:
        sim.set_hemodynamics(HemoParams(), baseline_hz=10.0, sample_every=25)
        g1 = sim.advance(200)
        g2 = sim.advance(200)
        st_gpu = sim.hemo_state()
    rs = RefSim(net, opt)
    r1, r2 = rs.advance(200), rs.advance(200)
    assert np.array_equal(g1.rates.counts, r1.rates) and np.array_equal(g2.rates.counts, r2.rates)
    for g, r in ((g1, r1), (g2, r2)):  # RateSeries::voxel_counts (stats.cpp:193-201)
        vc = np.zeros((r.rates.shape[1], net.tables.n_voxels), np.uint32)
        for u, unit in enumerate(units):
            vc[:, unit["voxel"]] += r.rates[u]
        assert np.array_equal(g.voxel_counts, vc)
    st = np.tile([0.0, 1.0, 1.0, 1.0], (net.tables.n_voxels, 1))
    b1 = ref_window_bold(HemoParams(), r1.rates, units["voxel"], vox_n, 1e-3, 10.0, 25, st)
    b2 = ref_window_bold(HemoParams(), r2.rates, units["voxel"], vox_n, 1e-3, 10.0, 25, st)
    assert g1.bold.shape == b1.shape == (8, net.tables.n_voxels)
    assert np.abs(b1).max() > 1e-5  # the drive moved the model (BOLD rises over seconds)
    assert close(g1.bold, b1) and close(g2.bold, b2)
    assert close(np.stack([st_gpu["s"], st_gpu["f"], st_gpu["v"], st_gpu["q"]], 1), st)


def test_engine_bold_validation():
    net = RefNet(make_config(seed=3, voxels=3, npv=50, k_in=5))
    with SimInstance(net.tables, SimOptions(steps=10)) as sim:
        with pytest.raises(ConfigError, match="alpha"):
            sim.set_hemodynamics(HemoParams(alpha=0.0))
        with pytest.raises(ConfigError, match="baseline_hz"):
            sim.set_hemodynamics(HemoParams(), baseline_hz=0.0)
        with pytest.raises(ConfigError, match="sample_every"):
            sim.set_hemodynamics(HemoParams(), sample_every=0)
        sim.set_hemodynamics(HemoParams(), baseline_hz=5.0, sample_every=3)
        r = sim.advance(10)
        assert r.bold.shape == (3, 3)
