"""CPU checks of the assimilation host loop (assim.py) against the
reference's own pieces (assim.cpp through oracle/_ref): the EnSRF update,
Pearson r, the prior ensemble, and the exact conductance sampler."""
import math

import numpy as np
import pytest

from paper_2308_01241_b200 import assim, netgen
from paper_2308_01241_b200.engine import ConfigError
from refnet import ref_ensrf, ref_sample_conductances


def test_ensrf_zero_innovation_keeps_the_mean_and_inflates():
    # assim.hpp:78-80: zero innovation leaves the ensemble mean unchanged exactly
    rng = np.random.default_rng(1)
    ens = [list(rng.normal(size=3)) for _ in range(6)]
    fc = [list(rng.normal(size=4)) for _ in range(6)]
    mean_fc = [sum(f[o] for f in fc) / 6 for o in range(4)]
    before = [sum(e[c] for e in ens) / 6 for c in range(3)]
    assim.ensrf_update(ens, fc, mean_fc, 1e-6, 1.0, 0.0)
    after = [sum(e[c] for e in ens) / 6 for c in range(3)]
    assert np.allclose(before, after, rtol=0, atol=1e-12)


def test_ensrf_degenerate_ensemble_reseeds_spread_and_validates():
    ens = [[0.5] for _ in range(4)]
    fc = [[1.0] for _ in range(4)]
    assim.ensrf_update(ens, fc, [1.0], 1.0, 1.05, 1e-3)
    sd = np.std([e[0] for e in ens], ddof=1)
    assert sd > 0 and abs(np.mean([e[0] for e in ens]) - 0.5) < 1e-12
    with pytest.raises(ConfigError):
        assim.ensrf_update([[0.0]], [[0.0]], [0.0], 1.0, 1.0, 0.0)


def test_pearson_and_validation():
    assert assim.pearson([1, 2, 3], [2, 4, 6]) == pytest.approx(1.0)
    assert assim.pearson([1, 1, 1], [1, 2, 3]) == 0.0
    with pytest.raises(ConfigError, match="members"):
        assim.validate_assim(assim.AssimOptions(members=1, targets=[assim.AssimTarget()]))
    with pytest.raises(ConfigError, match="targets"):
        assim.validate_assim(assim.AssimOptions())


def test_exact_conductances_equal_the_reference():
    # netgen.cpp:318-329 through oracle/_ref, per-member salts of assim.cpp:98-103
    for member in (-1, 0, 3):
        salt = netgen.mix_key((member + 1) & (2**64 - 1), 5)
        v = netgen.sample_conductances_exact(3, salt, 2, 1, -0.5, 0.2, 2000)
        assert v.dtype == np.float32
        assert np.array_equal(v, ref_sample_conductances(3, salt, 2, 1, -0.5, 0.2, 2000))


@pytest.mark.parametrize("m,p,q", [(4, 2, 3), (8, 3, 20), (16, 1, 200)])
def test_ensrf_equals_the_reference_bit_for_bit(m, p, q):
    rng = np.random.default_rng(m * 100 + q)
    ens = rng.normal(-1.0, 0.3, size=(m, p))
    fc = rng.normal(0.01, 0.004, size=(m, q))
    obs = rng.normal(0.01, 0.004, size=q)
    mine = [list(r) for r in ens]
    assim.ensrf_update(mine, [list(r) for r in fc], list(obs), 4e-8, 1.05, 1e-3)
    assert np.array_equal(np.array(mine), ref_ensrf(ens, fc, obs, 4e-8, 1.05, 1e-3))
