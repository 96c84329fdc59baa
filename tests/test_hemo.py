"""CPU checks of the BOLD-proxy readout harness: the reference's own
hemodynamics (hemo.cpp through oracle/_ref) against the known answers of
/root/reference/proj/tests/test_hemo.cpp, so the checker the GPU tests use is
pinned, plus the host-side parameter mirror (hemo.hpp:10-23)."""
import numpy as np
import pytest

from paper_2308_01241_b200.engine import HEMO_STATE_DTYPE, ConfigError, HemoParams, SimError, hemo_rest
from refnet import ref_bold_from_drive, ref_window_bold


# test_hemo.cpp:14-33
def test_default_parameters_and_derived_factors():
    p = HemoParams()
    assert p.k1() == pytest.approx(2.38)
    assert p.k2() == 2.0
    assert p.k3() == pytest.approx(0.48)
    st = hemo_rest(3)
    assert st.dtype == HEMO_STATE_DTYPE and st["f"].tolist() == [1.0] * 3 and st["s"].sum() == 0


# test_hemo.cpp:35-45
def test_reference_rest_is_a_fixed_point():
    st = np.array([0.0, 1.0, 1.0, 1.0])
    b = ref_bold_from_drive(HemoParams(), np.zeros(5000), 0.001, 1, st)
    assert np.all(b == 0.0) and st.tolist() == [0.0, 1.0, 1.0, 1.0]


# test_hemo.cpp:47-61: one Euler step from (0.1, 1.2, 1.1, 0.9), drive 0.5, dt 10 ms
def test_reference_one_euler_step():
    st = np.array([0.1, 1.2, 1.1, 0.9])
    b = ref_bold_from_drive(HemoParams(), [0.5], 0.01, 1, st)
    assert st[0] == pytest.approx(0.10353000000000001, rel=1e-14)
    assert st[1] == pytest.approx(1.201, rel=1e-14)
    assert st[2] == pytest.approx(1.0985004891109096, rel=1e-12)
    assert st[3] == pytest.approx(0.8992950357636457, rel=1e-12)
    assert b[0] == pytest.approx(0.01110167448431187, rel=1e-10)


# test_hemo.cpp:108-134 and 136-141
def test_reference_sampling_carry_and_errors():
    z = np.full(1000, 0.7)
    sampled = ref_bold_from_drive(HemoParams(), z, 0.001, 100)
    dense = ref_bold_from_drive(HemoParams(), z, 0.001, 1)
    assert sampled[0] == dense[99] and sampled[9] == dense[999]
    with pytest.raises(ConfigError):
        ref_bold_from_drive(HemoParams(), z, 0.001, 0)
    with pytest.raises(SimError):
        ref_bold_from_drive(HemoParams(), [0.0], 0.001, 1, np.array([np.inf, 1.0, 1.0, 1.0]))


# window_bold (assim.cpp:51-71) == bold_from_drive on the voxel drive
def test_reference_window_bold_is_bold_from_drive_of_the_voxel_drive():
    rng = np.random.default_rng(5)
    counts = rng.integers(0, 40, size=(4, 300)).astype(np.uint32)  # 4 units, 2 voxels
    unit_voxel = np.array([0, 0, 1, 1])
    vox_n = np.array([500, 700], np.uint64)
    st = np.tile([0.0, 1.0, 1.0, 1.0], (2, 1))
    b = ref_window_bold(HemoParams(), counts, unit_voxel, vox_n, 0.001, 10.0, 30, st)
    for v in range(2):
        c = counts[unit_voxel == v].sum(axis=0)
        z = c / (float(vox_n[v]) * 0.001) / 10.0
        sv = np.array([0.0, 1.0, 1.0, 1.0])
        assert np.array_equal(ref_bold_from_drive(HemoParams(), z, 0.001, 30, sv), b[:, v])
        assert np.array_equal(sv, st[v])
