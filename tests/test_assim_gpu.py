"""Twin-experiment assimilation with device members (assim.py) against the
reference's own assimilate / run_forward_bold (assim.cpp via oracle/_ref) on
the same network.  Members' spikes are the reference's; BOLD differs only by
pow() ulps (see test_hemo_gpu.py), so forecasts, filter statistics and the
posterior agree to 1e-9 relative."""
import numpy as np
import pytest

from paper_2308_01241_b200 import assim
from paper_2308_01241_b200.engine import SimInstance, SimOptions
from refnet import RefNet, make_config, ref_assimilate, ref_forward_bold, ref_unit_pop

pytestmark = pytest.mark.gpu


def setup():
    net = RefNet(make_config(seed=11, voxels=3, npv=300, k_in=30, rho=0.3, ou_mean=350.0,
                             ou_sigma=150.0))
    opts = assim.AssimOptions(members=4, windows=4, window_steps=150, obs_noise_sd=2e-4,
                              baseline_hz=10.0, seed=5,
                              targets=[assim.AssimTarget(0, 0), assim.AssimTarget(2, 0)])
    loc, scale = [], []
    for t in opts.targets:
        gl, gs = ref_unit_pop(net, t.unit)
        loc.append(gl[t.receptor])
        scale.append(gs[t.receptor])
    return net, opts, loc, scale


def close(a, b, rel):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and np.all(np.abs(a - b) <= rel * np.abs(b) + 1e-14)


def test_forward_bold_and_assimilation_match_the_reference():
    net, opts, loc, scale = setup()
    truth_params = [x + 0.3 for x in loc]
    with SimInstance(net.tables, SimOptions(steps=opts.window_steps, record_raster=False)) as donor:
        units = net.tables.units
        fwd = assim.run_forward_bold(donor, units, opts, opts.windows, truth_params, scale)
        ref_fwd = ref_forward_bold(net, opts, opts.windows, truth_params)
        assert np.abs(ref_fwd).max() > 1e-5
        assert close(fwd, ref_fwd, 1e-12)
        plain = assim.run_forward_bold(donor, units, opts, 2)
        assert close(plain, ref_forward_bold(net, opts, 2), 1e-12)
        res = assim.assimilate(donor, units, ref_fwd, opts, loc, scale)
    stats, fmean, fspread, div = ref_assimilate(net, ref_fwd, opts)
    assert len(res.windows) == len(stats) == opts.windows and not res.diverged and div == 0
    mine = np.array([[w.window, w.innovation_rms, w.pearson_r, w.mean_spread, *w.target_mean]
                     for w in res.windows])
    assert close(mine, stats, 1e-9)
    assert close(res.final_mean, fmean, 1e-9) and close(res.final_spread, fspread, 1e-9)
