"""Parity in the regime the benchmark times ("what's weak" 1).

bench.py's config-2 line runs K = 1000 rows at the calibrated ~10 Hz point
(g_location[AMPA] = -2.3, ou_mean = 275) with dt = 1 ms, one-spike dynamic
chunks (ch_max = 1, taken when in-degree per L2 block >= 512) and tables
generated on the device; config 3 runs K = 500 on a lognormal-voxel-size
DTI-like connectome with L2-blocked delivery (n_blocks > 1, 1024-entry
stages, 32-spike chunks).  These tests run the UNMODIFIED reference engine
(oracle/_ref, SimInstance::advance, engine.cpp:763-827) and the CUDA engine on
byte-identical networks in those regimes and require:

* rasters, rate series, FLOP tallies and the final membrane state bit-exact
  (north_star: "spike rasters must be bit-exact");
* per-voxel firing rates over 1 s of biological time within 1 % (north_star;
  implied by the above, asserted explicitly);
* the schedule actually taken is the benchmark's (checked through
  vxb_schedule_info, so a silent change of path cannot pass unnoticed).

Network sizes are the largest slices the reference builds in well under a
minute: 12 voxels x 10 000 neurons at K = 1000 (1.2e8 synapses — the network
bench.py's CPU arm times) and a 200-voxel DTI-like slice of 2e5 neurons at
K = 500.
"""
import os

import numpy as np
import pytest

from paper_2308_01241_b200 import netgen
from paper_2308_01241_b200.engine import SimOptions
from refnet import RefNet, RefSim

pytestmark = pytest.mark.gpu


def _voxel_rates(counts, units, n_voxels, steps, dt_ms):
    """Per-voxel firing rate (Hz) from RateSeries counts [unit][step]."""
    spikes = np.zeros(n_voxels, np.float64)
    neurons = np.zeros(n_voxels, np.float64)
    np.add.at(spikes, units["voxel"], counts.sum(axis=1))
    np.add.at(neurons, units["voxel"], units["neurons"])
    return spikes / np.maximum(neurons, 1) / (steps * dt_ms * 1e-3)


def _compare(cfg, steps, chunks, expect, tuning=None, monkeypatch=None):
    if tuning:
        monkeypatch.setenv("VXB_TUNING", "1")
        for k, v in tuning.items():
            monkeypatch.setenv(k, v)
    dt = cfg["dt_ms"]
    # CUDA engine on the device-generated tables: exactly bench.py's path
    net = netgen.build_network(cfg)
    opt = SimOptions(steps=steps, dt_ms=dt, record_raster=True, record_timings=False)
    with netgen.GeneratedSimInstance(net, opt) as sim:
        sched = sim.schedule_info()
        res = [sim.advance(c) for c in chunks]
        snap = [sim.membrane_snapshot(w) for w in range(sim.workers)]
    for k, v in expect.items():
        assert sched[k] == v, (k, sched)
    # the reference engine on the reference pipeline's tables (same config)
    ref_net = RefNet(cfg)
    rs = RefSim(ref_net, SimOptions(steps=steps, dt_ms=dt, record_raster=True,
                                    record_timings=False),
                scheduler="threads" if cfg.get("workers", 1) > 1 else "loopback")
    ref = rs.advance(steps)
    # rasters: (step, worker, local, gid), in the reference's order
    g_r = np.concatenate([r.raster for r in res])
    assert g_r.shape == ref.raster.shape
    for f in ("step", "worker", "local", "gid"):
        assert np.array_equal(g_r[f], ref.raster[f]), f
    counts = np.concatenate([r.rates.counts for r in res], axis=1)
    assert np.array_equal(counts, ref.rates)
    fl = {k: sum(r.flops[k] for r in res) for k in res[0].flops}
    assert fl == ref.flops
    for w in range(len(snap)):
        assert np.array_equal(snap[w], rs.membrane_snapshot(w)), w
    units = ref_net.tables.units
    vr_gpu = _voxel_rates(counts, units, ref_net.tables.n_voxels, steps, dt)
    vr_ref = _voxel_rates(ref.rates, units, ref_net.tables.n_voxels, steps, dt)
    assert np.all(np.abs(vr_gpu - vr_ref) <= 0.01 * np.maximum(vr_ref, 1e-12))
    return ref, vr_ref, sched


@pytest.mark.parametrize("path", ["tile", "l2"])
def test_config2_regime_ring12_k1000_one_bio_second(monkeypatch, path):
    """Config 2's operating point on a 12-voxel ring (1.2e8 synapses), 1000
    steps of dt = 1 ms in two advances, generated tables: the SM-tile path
    bench.py takes on one GPU, and the l2_atomic path (one-spike chunks)."""
    import bench
    cfg = bench.workload_cfg(voxels=12)
    expect = ({"path": "sm_tile"} if path == "tile" else
              {"path": "l2_atomic", "l2_blocks": 1, "dynamic_deal": 1, "ch_max": 1})
    ref, vr, _ = _compare(cfg, 1000, [400, 600], expect, tuning={"VXB_PATH": path},
                          monkeypatch=monkeypatch)
    rate = ref.total_spikes / (120_000 * 1.0)
    assert 7.0 < rate < 13.0, rate  # the calibrated ~10 Hz point
    assert vr.min() > 0


def _host_gb():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30
    except (ValueError, OSError):
        return 0.0


@pytest.mark.skipif(_host_gb() < 150 and not os.environ.get("VXB_FULL_PARITY"),
                    reason="needs >= 150 GB of host memory for the reference's 1e9-synapse tables")
def test_config2_full_size_300_steps():
    """Config 2 itself — the benchmark's 1M neurons, K = 1000 (1e9 synapses),
    10 Hz point — 300 steps in two advances on the SM-tile path, against the
    reference engine on the reference pipeline's tables: raster, rates,
    FLOPs and the final membrane state bit-exact, per-voxel rates within 1 %."""
    import bench
    cfg = bench.workload_cfg()
    ref, vr, _ = _compare(cfg, 300, [100, 200], {"path": "sm_tile"})
    rate = ref.total_spikes / (1_000_000 * 0.3)
    assert 7.0 < rate < 13.0, rate
    assert vr.min() > 0


def test_config3_regime_dti_slice_l2_blocked(monkeypatch, tmp_path):
    """Config 3's shape: 200-voxel DTI-like connectome with lognormal voxel
    sizes (2e5 neurons), K = 500 at the 10 Hz point, 2 workers (greedy
    partition) on one device, delivery split into 4 L2 blocks with the
    default 1024-entry stages and 32-spike chunks."""
    import bench
    path = tmp_path / "dti200.txt"
    netgen.write_connectome_file(netgen.dti_like_connectome(total_neurons=200_000), path)
    ampa, ou = bench.K500_POINTS[10]
    cfg = {"seed": bench.SEED, "dt_ms": 1.0, "steps": 400, "workers": 2,
           "scheduler": "loopback",
           "connectome": {"kind": "file", "path": str(path)},
           "partition": {"method": "greedy"},
           "regions": {"subcortex": {"k_in": 500, "g_location": [ampa] + bench.G_LOC_10HZ[1:],
                                     "ou_mean": ou}}}
    ref, vr, sched = _compare(cfg, 400, [150, 250],
                              {"path": "l2_atomic", "l2_blocks": 4, "stage_entries": 1024,
                               "ch_max": 32},
                              tuning={"VXB_PATH": "l2", "VXB_BLOCK_NEURONS": "50000"},
                              monkeypatch=monkeypatch)
    assert ref.total_spikes > 100_000


def test_config3_slice_sm_tile_path(monkeypatch, tmp_path):
    """The same DTI-like slice shape (lognormal voxel sizes, K = 500, greedy
    2-worker partition) on the SM-tile path: short, irregular (source,
    tile) segments."""
    import bench
    path = tmp_path / "dti200.txt"
    netgen.write_connectome_file(netgen.dti_like_connectome(total_neurons=200_000), path)
    ampa, ou = bench.K500_POINTS[10]
    cfg = {"seed": bench.SEED, "dt_ms": 1.0, "steps": 300, "workers": 2,
           "scheduler": "loopback",
           "connectome": {"kind": "file", "path": str(path)},
           "partition": {"method": "greedy"},
           "regions": {"subcortex": {"k_in": 500, "g_location": [ampa] + bench.G_LOC_10HZ[1:],
                                     "ou_mean": ou}}}
    ref, _, _ = _compare(cfg, 300, [100, 200], {"path": "sm_tile"}, tuning={"VXB_PATH": "tile"},
                         monkeypatch=monkeypatch)
    assert ref.total_spikes > 100_000


def test_config3_slice_multipass_tiles(monkeypatch, tmp_path):
    """The DTI-like slice on the several-tiles-per-SM kernel (tile_mp_kernel,
    the configs-3-5 path): 256-neuron tiles, so ~5 passes per CTA, and short
    segments consumed one queue item per lane."""
    import bench
    path = tmp_path / "dti200.txt"
    netgen.write_connectome_file(netgen.dti_like_connectome(total_neurons=200_000), path)
    ampa, ou = bench.K500_POINTS[10]
    cfg = {"seed": bench.SEED, "dt_ms": 1.0, "steps": 300, "workers": 2,
           "scheduler": "loopback",
           "connectome": {"kind": "file", "path": str(path)},
           "partition": {"method": "greedy"},
           "regions": {"subcortex": {"k_in": 500, "g_location": [ampa] + bench.G_LOC_10HZ[1:],
                                     "ou_mean": ou}}}
    ref, _, sched = _compare(cfg, 300, [120, 180], {"path": "sm_tile", "kernel": "vxb::tile_mp_kernel",
                                                    "item_per": "lane"},
                             tuning={"VXB_PATH": "tile", "VXB_TILE_PER": "256"},
                             monkeypatch=monkeypatch)
    assert sched["passes"] >= 5 and ref.total_spikes > 100_000
