"""GPU parity tests: the CUDA engine (through the C ABI) against the reference.

Each case mirrors a TEST_CASE of /root/reference/proj/tests/test_engine.cpp and
compares the B200 engine with the UNMODIFIED reference engine
(oracle/_ref/libvoxsim_ref.so) or the C restatement (oracle/voxsim_oracle.c)
on byte-identical tables.  Integer/index results must be bit-exact; float
traces are compared bitwise (the north-star tolerance, 1e-5 relative, is the
fallback stated where used).
"""
import numpy as np
import pytest

from paper_2308_01241_b200.engine import (ConfigError, ForcedSpike, Injection, SimError,
                                          SimInstance, SimOptions, run_simulation)
from refnet import OracleSim, RefNet, RefSim, make_config, raster_set

pytestmark = pytest.mark.gpu


def quiet_cfg(**kw):
    return make_config(ou_mean=0.0, ou_sigma=0.0, **kw)


def hot_cfg(**kw):
    return make_config(ou_mean=400.0, ou_sigma=150.0, **kw)


def gpu_run(tables, opt, steps=None):
    with SimInstance(tables, opt) as sim:
        r = sim.advance(opt.steps if steps is None else steps)
        snaps = [sim.membrane_snapshot(w) for w in range(sim.workers)]
    return r, snaps


def assert_same(gpu, ref, probes=True, same_partition=True):
    assert gpu.total_spikes == ref.total_spikes
    assert raster_set(gpu.raster) == raster_set(ref.raster)
    assert np.array_equal(gpu.rates.counts, ref.rates)
    if probes and ref.probe_v.size:
        assert np.array_equal(np.stack([p.v for p in gpu.probes]), ref.probe_v)
        assert np.array_equal(np.stack([p.i_syn for p in gpu.probes]), ref.probe_i)
    if same_partition:
        assert gpu.flops == ref.flops
    else:  # inner/outer split follows the worker partition; the sum does not
        g, r = dict(gpu.flops), dict(ref.flops)
        assert g.pop("gating_inner") + g.pop("gating_outer") == \
            r.pop("gating_inner") + r.pop("gating_outer")
        assert g == r


# test_engine.cpp:107-201
def test_matches_reference_bit_for_bit_six_neurons():
    net = RefNet(make_config(seed=91, voxels=1, npv=6, k_in=2))
    opt = SimOptions(steps=150, probe_gids=list(range(6)))
    gpu, snaps = gpu_run(net.tables, opt)
    rs = RefSim(net, opt)
    ref = rs.advance(150)
    assert ref.total_spikes > 0
    assert_same(gpu, ref)
    assert np.array_equal(snaps[0], rs.membrane_snapshot(0))


@pytest.mark.parametrize("workers", [1, 2, 3])
def test_matches_reference_ring(workers):
    net = RefNet(make_config(seed=5, voxels=3, npv=60, k_in=8, rho=0.4), even_workers=workers)
    opt = SimOptions(steps=120, probe_gids=[7, 179, 60])
    gpu, snaps = gpu_run(net.tables, opt)
    rs = RefSim(net, opt)
    ref = rs.advance(120)
    assert ref.total_spikes > 0
    assert_same(gpu, ref)
    for w in range(workers):
        assert np.array_equal(snaps[w], rs.membrane_snapshot(w))


# Config 1 of BASELINE.json: 10k neurons, K=100, dt=0.1 ms, 1 s, seed 1.
def test_config1_one_bio_second():
    cfg = make_config(seed=1, voxels=1, npv=10000, k_in=100, dt_ms=0.1, steps=10000)
    net = RefNet(cfg)
    opt = SimOptions(steps=10000, dt_ms=0.1, probe_gids=[0, 4321, 9999])
    gpu, snaps = gpu_run(net.tables, opt)
    assert gpu.total_spikes == 33078  # survey golden
    rs = RefSim(net, opt)
    ref = rs.advance(10000)
    assert_same(gpu, ref)
    assert np.array_equal(snaps[0], rs.membrane_snapshot(0))


# test_engine.cpp:203-246
def test_spike_delivery_lags_one_step():
    net = RefNet(quiet_cfg(seed=17, voxels=1, npv=10, k_in=3))
    w0 = net.tables.workers[0]
    rb, syn = w0.row_base, w0.synapses
    target = next(t for t in range(10)
                  if (syn["src_local"][rb[t]:rb[t + 1]] == 0).any())
    gid_t = int(w0.neurons["gid"][target])
    base = SimOptions(steps=12, probe_gids=[gid_t])
    forced = SimOptions(steps=12, probe_gids=[gid_t],
                        forced_spikes=[ForcedSpike(5, int(w0.neurons["gid"][0]))])
    q = run_simulation(net.tables, base)
    s = run_simulation(net.tables, forced)
    qp, sp = q.probes[0], s.probes[0]
    assert np.array_equal(sp.i_syn[:6], qp.i_syn[:6])
    assert np.array_equal(sp.v[:6], qp.v[:6])
    assert sp.i_syn[6] != qp.i_syn[6]
    assert sp.v[6] == qp.v[6]
    assert sp.v[7] != qp.v[7]
    assert (5, int(w0.neurons["gid"][0])) in raster_set(s.raster)
    assert s.total_spikes == q.total_spikes + 1
    ref = RefSim(net, forced).advance(12)
    assert_same(s, ref)


# test_engine.cpp:248-261
def test_forced_spike_on_fired_neuron_is_dropped():
    net = RefNet(hot_cfg(seed=3, voxels=1, npv=8, k_in=2))
    opt = SimOptions(steps=30)
    base = run_simulation(net.tables, opt)
    assert base.total_spikes > 0
    ev = base.raster[0]
    opt2 = SimOptions(steps=30, forced_spikes=[ForcedSpike(int(ev["step"]), int(ev["gid"]))])
    forced = run_simulation(net.tables, opt2)
    assert forced.total_spikes == base.total_spikes
    assert raster_set(forced.raster) == raster_set(base.raster)


# test_engine.cpp:263-301
def test_piecewise_advance_equals_whole():
    net = RefNet(make_config(seed=23, voxels=3, npv=40, k_in=5, rho=0.3))
    opt = SimOptions(steps=90, probe_gids=[0, 41, 100])
    with SimInstance(net.tables, opt) as whole:
        rw = whole.advance(90)
        snap_w = whole.membrane_snapshot(0)
    with SimInstance(net.tables, opt) as pieces:
        r1, r2, r3 = pieces.advance(30), pieces.advance(45), pieces.advance(15)
        assert pieces.current_step() == 90
        snap_p = pieces.membrane_snapshot(0)
    assert r1.steps_done == 30 and r2.steps_done == 45
    allr = raster_set(r1.raster) + raster_set(r2.raster) + raster_set(r3.raster)
    assert sorted(allr) == raster_set(rw.raster)
    assert r1.total_spikes + r2.total_spikes + r3.total_spikes == rw.total_spikes
    for p in range(3):
        v = np.concatenate([r.probes[p].v for r in (r1, r2, r3)])
        i = np.concatenate([r.probes[p].i_syn for r in (r1, r2, r3)])
        assert np.array_equal(v, rw.probes[p].v)
        assert np.array_equal(i, rw.probes[p].i_syn)
    assert np.array_equal(snap_w, snap_p)
    ref = RefSim(net, opt).advance(90)
    assert_same(rw, ref)


# test_engine.cpp:322-358
def test_results_independent_of_partition():
    cfg = make_config(seed=44, voxels=3, npv=50, k_in=6, rho=0.5)
    opt = SimOptions(steps=100, probe_gids=[0, 60, 149])
    results = [run_simulation(RefNet(cfg, even_workers=w).tables, opt) for w in (1, 2, 3)]
    for r in results[1:]:
        assert r.total_spikes == results[0].total_spikes
        assert raster_set(r.raster) == raster_set(results[0].raster)
        for p in range(3):
            assert np.array_equal(r.probes[p].v, results[0].probes[p].v)
            assert np.array_equal(r.probes[p].i_syn, results[0].probes[p].i_syn)
    assert results[0].total_spikes > 0
    assert results[2].flops["gating_outer"] > 0


# test_engine.cpp:360-387
def test_flop_accounting_is_exact():
    n, steps = 30, 50
    net = RefNet(quiet_cfg(seed=7, voxels=1, npv=n, k_in=3))
    res = run_simulation(net.tables, SimOptions(steps=steps))
    assert res.total_spikes == 0
    assert res.flops["membrane"] == 6 * n * steps
    assert res.flops["gating_decay"] == 12 * n * steps
    assert res.flops["current"] == 16 * n * steps
    assert res.flops["gating_inner"] == 0 and res.flops["gating_outer"] == 0
    w0 = net.tables.workers[0]
    fanout = int((w0.synapses["src_local"] == 0).sum())
    res = run_simulation(net.tables, SimOptions(
        steps=steps, forced_spikes=[ForcedSpike(10, int(w0.neurons["gid"][0]))]))
    assert res.total_spikes == 1
    assert res.flops["gating_inner"] == 2 * fanout
    assert res.flops["gating_outer"] == 0


# test_engine.cpp:389-405 (ring-mode spike log: raster off)
def test_rates_recorded_with_raster_disabled():
    net = RefNet(hot_cfg(seed=2, voxels=1, npv=40, k_in=4))
    opt = SimOptions(steps=80, record_raster=False)
    res = run_simulation(net.tables, opt)
    assert res.raster.size == 0
    assert res.total_spikes > 0
    assert int(res.rates.counts.sum()) == res.total_spikes
    hz = res.total_spikes / (80 * 0.001) / 40
    assert abs(res.rates.network_mean_hz(0) - hz) <= 1e-9 * hz
    ref = RefSim(net, opt).advance(80)
    assert np.array_equal(res.rates.counts, ref.rates)
    assert res.flops == ref.flops


# test_engine.cpp:467-500
def test_injection_drives_only_its_voxel():
    net = RefNet(quiet_cfg(seed=8, voxels=3, npv=30, k_in=4))
    opt = SimOptions(steps=60, injections=[Injection(10, 50, 1, 1000.0)])
    res = run_simulation(net.tables, opt)
    assert res.total_spikes > 0
    units = net.tables.units
    for ev in res.raster:
        u = np.searchsorted(units["gid_base"], ev["gid"], side="right") - 1
        assert units["voxel"][u] == 1
        assert 10 <= ev["step"] < 55
    ref = RefSim(net, opt).advance(60)
    assert_same(res, ref)
    with pytest.raises(ConfigError):
        run_simulation(net.tables, SimOptions(steps=10, injections=[Injection(0, 5, 99, 1.0)]))
    with pytest.raises(ConfigError):
        run_simulation(net.tables, SimOptions(steps=10, injections=[Injection(8, 2, 0, 1.0)]))
    with pytest.raises(SimError, match="membrane potential diverged"):
        run_simulation(net.tables, SimOptions(steps=10,
                                              injections=[Injection(0, 10, 0, float("inf"))]))


def test_failed_instance_rejects_advance():
    net = RefNet(quiet_cfg(seed=8, voxels=3, npv=30, k_in=4))
    with SimInstance(net.tables, SimOptions(
            steps=10, injections=[Injection(0, 10, 0, float("inf"))])) as sim:
        with pytest.raises(SimError):
            sim.advance(10)
        with pytest.raises(SimError, match="failed state"):
            sim.advance(1)


# test_engine.cpp:502-537
def test_conductance_override():
    net = RefNet(quiet_cfg(seed=12, voxels=1, npv=20, k_in=2))
    w0 = net.tables.workers[0]
    opt = SimOptions(steps=20, probe_gids=[0, 5, 19],
                     forced_spikes=[ForcedSpike(3, int(w0.neurons["gid"][2])),
                                    ForcedSpike(4, int(w0.neurons["gid"][7]))])
    with SimInstance(net.tables, opt) as sim:
        for u in range(net.tables.units.shape[0]):
            nu = int(net.tables.units["neurons"][u])
            for rc in range(4):
                sim.set_conductances(u, rc, np.zeros(nu, np.float32))
        res = sim.advance(20)
    for p in res.probes:
        assert (p.i_syn == 0.0).all()
    assert res.total_spikes == 2
    with SimInstance(net.tables, SimOptions(steps=5)) as sim:
        n0 = int(net.tables.units["neurons"][0])
        with pytest.raises(ConfigError):
            sim.set_conductances(99, 0, np.ones(4, np.float32))
        with pytest.raises(ConfigError):
            sim.set_conductances(0, 7, np.ones(n0, np.float32))
        with pytest.raises(ConfigError):
            sim.set_conductances(0, 0, np.ones(n0 + 1, np.float32))
        with pytest.raises(ConfigError):
            sim.set_conductances(0, 0, -np.ones(n0, np.float32))
        with pytest.raises(ConfigError):
            sim.membrane_snapshot(5)


def test_conductance_override_matches_reference():
    net = RefNet(hot_cfg(seed=13, voxels=3, npv=50, k_in=6, rho=0.2))
    opt = SimOptions(steps=40, probe_gids=[3, 77])
    vals = np.linspace(0.0, 3.0, int(net.tables.units["neurons"][1])).astype(np.float32)
    rs = RefSim(net, opt)
    rs.set_conductances(1, 2, vals)
    ref = rs.advance(40)
    with SimInstance(net.tables, opt) as sim:
        sim.set_conductances(1, 2, vals)
        gpu = sim.advance(40)
    assert_same(gpu, ref)


def test_conductance_staging_matches_reference():
    """set_conductances is staged on the host and applied by the next advance;
    repeated sets, sets between advances and the reference's prefix-written
    error path (engine.cpp:839-843) must all land exactly as in the reference."""
    net = RefNet(hot_cfg(seed=17, voxels=3, npv=40, k_in=6, rho=0.2))
    opt = SimOptions(steps=30, probe_gids=[5, 60, 100])
    nus = [int(x) for x in net.tables.units["neurons"]]
    rng = np.random.default_rng(4)
    bad = rng.uniform(0.0, 2.0, nus[0]).astype(np.float32)
    bad[nus[0] // 2] = np.nan  # prefix before the NaN is written, then ConfigError

    def script(sim):
        out = []
        sim.set_conductances(1, 0, rng_vals(1, 0))
        sim.set_conductances(1, 0, rng_vals(1, 1))  # overwrites the first set
        sim.set_conductances(2, 3, rng_vals(2, 2))
        with pytest.raises(ConfigError):
            sim.set_conductances(0, 1, bad)
        out.append(sim.advance(15))
        sim.set_conductances(2, 3, rng_vals(2, 3))
        sim.set_conductances(0, 0, rng_vals(0, 4))
        out.append(sim.advance(15))
        return out

    def rng_vals(u, k):
        return np.random.default_rng(100 + k).uniform(0.0, 2.5, nus[u]).astype(np.float32)

    ref = script(RefSim(net, opt))
    with SimInstance(net.tables, opt) as sim:
        gpu = script(sim)
    for g, r in zip(gpu, ref):
        assert_same(g, r)


# test_engine.cpp:539-558
def test_option_validation():
    net = RefNet(quiet_cfg(seed=1, voxels=1, npv=10, k_in=2))
    bad = [dict(dt_ms=0.0), dict(scheduler="mpi"), dict(workers_per_node=0),
           dict(transport="rdma")]
    for kw in bad:
        with pytest.raises(ConfigError):
            run_simulation(net.tables, SimOptions(steps=5, **kw))
    with pytest.raises(SimError):
        run_simulation(net.tables, SimOptions(steps=5, probe_gids=[100000]))


# test_engine.cpp:560-570
def test_identical_runs_reproduce():
    net = RefNet(make_config(seed=31, voxels=3, npv=50, k_in=6, rho=0.3), even_workers=2)
    opt = SimOptions(steps=70, probe_gids=[10])
    a, b = run_simulation(net.tables, opt), run_simulation(net.tables, opt)
    assert a.total_spikes == b.total_spikes
    assert raster_set(a.raster) == raster_set(b.raster)
    assert np.array_equal(a.probes[0].v, b.probes[0].v)
    assert a.flops == b.flops


def test_zero_steps_is_a_noop():
    net = RefNet(make_config(seed=3, voxels=1, npv=20, k_in=3))
    with SimInstance(net.tables, SimOptions(steps=0)) as sim:
        r = sim.advance(0)
        assert r.steps_done == 0 and r.total_spikes == 0 and sim.current_step() == 0


def test_wide_accumulators_on_signed_weights():
    """Negative / oversized Q16 weights force the four-int64 pending layout;
    checked against the C oracle on the same (edited) tables."""
    net = RefNet(hot_cfg(seed=21, voxels=1, npv=80, k_in=10))
    t = net.tables
    syn = t.workers[0].synapses
    syn["wq_fast"][::3] = -syn["wq_fast"][::3]
    opt = SimOptions(steps=60, probe_gids=[1, 40])
    gpu, snaps = gpu_run(t, opt)
    orc = OracleSim(t, opt)
    ref = orc.advance(60)
    assert_same(gpu, ref)
    assert np.array_equal(snaps[0], orc.membrane_snapshot(0))


def test_timings_rows_shape():
    net = RefNet(make_config(seed=6, voxels=3, npv=30, k_in=4, rho=0.4), even_workers=2)
    res = run_simulation(net.tables, SimOptions(steps=40))
    t = res.timings
    assert t.shape[0] == 80
    assert (t["step"] == np.arange(80) // 2).all()
    assert (t["worker"] == np.arange(80) % 2).all()
    assert (t["t"][:, 1] >= t["t"][:, 0]).all() and (t["t"][:, 2] >= t["t"][:, 1]).all()
    assert int(t["spikes"].sum()) == res.total_spikes
    off = run_simulation(net.tables, SimOptions(steps=10, record_timings=False))
    assert off.timings.size == 0


# acceptance.cpp:126-228 (criterion 1): 1e5 neurons / 1e7 synapses / 1000 steps,
# bit-identical raster, probes and final state for 1/2/4/8 worker tables.
@pytest.mark.slow
def test_acceptance_1_multi_worker_equivalence():
    def cfg(workers):
        c = make_config(seed=1401, voxels=100, npv=1000, k_in=100, rho=6 / 25, steps=1000,
                        workers=workers, partition="sequential" if workers == 1 else "greedy")
        return c
    probes = [i * 8321 + 17 for i in range(12)]
    opt = SimOptions(steps=1000, probe_gids=probes)
    ref_net = RefNet(cfg(1))
    assert ref_net.tables.synapse_count == 10_000_000
    rs = RefSim(ref_net, opt)
    ref = rs.advance(1000)
    assert ref.total_spikes == 500170  # survey golden
    ref_state = rs.membrane_snapshot(0)
    for workers in (1, 2, 4, 8):
        net = ref_net if workers == 1 else RefNet(cfg(workers))
        gpu, snaps = gpu_run(net.tables, opt)
        assert_same(gpu, ref, same_partition=workers == 1)
        state = np.zeros(ref_state.shape, np.float32)
        for w, s in enumerate(snaps):
            state[net.tables.workers[w].neurons["gid"]] = s
        assert np.array_equal(state, ref_state)


def set_path(monkeypatch, path):
    """tile / l2 / mp (several tiles per SM, 32-neuron tiles) / mp_lane (mp
    with one queue item per lane)."""
    monkeypatch.setenv("VXB_TUNING", "1")
    monkeypatch.setenv("VXB_PATH", "l2" if path == "l2" else "tile")
    if path.startswith("mp"):
        monkeypatch.setenv("VXB_TILE_PER", "32")
        monkeypatch.setenv("VXB_TILE_ITEMS", "1" if path == "mp_lane" else "0")


@pytest.mark.parametrize("path,dyn", [("l2", "0"), ("l2", "1"), ("tile", "1"), ("mp", "1"),
                                      ("mp_lane", "1")])
def test_static_and_dynamic_delivery_match_reference(monkeypatch, path, dyn):
    """Every delivery schedule is bit-exact (config 1 shape): the l2_atomic
    path's static round-robin rows (VXB_DYN=0) and block-major dynamic
    chunks, and the SM-tile path (shared-memory pending tiles)."""
    set_path(monkeypatch, path)
    monkeypatch.setenv("VXB_DYN", dyn)
    cfg = make_config(seed=1, voxels=1, npv=10000, k_in=100, dt_ms=0.1, steps=3000)
    net = RefNet(cfg)
    opt = SimOptions(steps=3000, dt_ms=0.1, probe_gids=[0, 4321, 9999])
    gpu, snaps = gpu_run(net.tables, opt)
    rs = RefSim(net, opt)
    ref = rs.advance(3000)
    assert_same(gpu, ref)
    assert np.array_equal(snaps[0], rs.membrane_snapshot(0))


def test_many_segments_global_parameter_table():
    """More parameter segments than fit in shared memory (600 units): the
    segment table stays in global memory and the cached/galloping lookup
    must still find every neuron's segment."""
    net = RefNet(hot_cfg(seed=23, voxels=300, npv=30, k_in=8, rho=0.3))
    assert net.tables.units.shape[0] > 256
    opt = SimOptions(steps=60, probe_gids=[0, 4444, 8999])
    gpu, snaps = gpu_run(net.tables, opt)
    rs = RefSim(net, opt)
    ref = rs.advance(60)
    assert ref.total_spikes > 0
    assert_same(gpu, ref)
    assert np.array_equal(snaps[0], rs.membrane_snapshot(0))


def test_l2_blocked_delivery_matches_reference(monkeypatch):
    """L2-blocked delivery (target-sorted rows, per-source block offsets,
    blocks delivered in order), forced on a small network with 2048-neuron
    blocks: bit-exact against the reference."""
    monkeypatch.setenv("VXB_TUNING", "1")
    monkeypatch.setenv("VXB_PATH", "l2")
    monkeypatch.setenv("VXB_BLOCK_NEURONS", "2048")
    net = RefNet(make_config(seed=1401, voxels=10, npv=1000, k_in=100, rho=6 / 25))
    opt = SimOptions(steps=300, probe_gids=[5, 5000, 9999])
    gpu, snaps = gpu_run(net.tables, opt)
    rs = RefSim(net, opt)
    ref = rs.advance(300)
    assert ref.total_spikes > 0
    assert_same(gpu, ref)
    assert np.array_equal(snaps[0], rs.membrane_snapshot(0))


def test_advance_without_forced_spikes_or_injection_after_one_with():
    """Forced spikes and injections are keyed by absolute step
    (engine.cpp:352-361, 389-398): an advance whose window holds none must
    not replay the previous advance's tables, and a longer later advance
    must not read past them."""
    net = RefNet(make_config(seed=29, voxels=3, npv=200, k_in=12, rho=0.3), even_workers=2)
    g = net.tables.workers[0].neurons["gid"]
    opt = SimOptions(steps=130, probe_gids=[int(g[3]), 450],
                     forced_spikes=[ForcedSpike(10, int(g[3])), ForcedSpike(40, int(g[7]))],
                     injections=[Injection(0, 50, 0, 120.0), Injection(20, 45, 1, -60.0)])
    with SimInstance(net.tables, opt) as sim:
        a = sim.advance(50)
        b = sim.advance(80)
        snaps = [sim.membrane_snapshot(w) for w in range(2)]
    rs = RefSim(net, opt)
    ra = rs.advance(50)
    rb = rs.advance(80)
    assert rb.total_spikes > 0
    assert_same(a, ra)
    assert_same(b, rb)
    for w in range(2):
        assert np.array_equal(snaps[w], rs.membrane_snapshot(w))


@pytest.mark.parametrize("path", ["tile", "l2", "mp", "mp_lane"])
def test_ring_multiworker_both_paths(monkeypatch, path):
    """3 workers on one device, both delivery paths, two advances: the
    SM-tile path (default for shards that fit on chip) and the l2_atomic
    path give the reference's results bit for bit."""
    set_path(monkeypatch, path)
    net = RefNet(hot_cfg(seed=31, voxels=5, npv=2000, k_in=40, rho=0.3), even_workers=3)
    opt = SimOptions(steps=150, probe_gids=[3, 1000, 9999])
    with SimInstance(net.tables, opt) as sim:
        info = sim.schedule_info()
        assert info["path"] == ("l2_atomic" if path == "l2" else "sm_tile")
        if path.startswith("mp"):
            assert info["kernel"] == "vxb::tile_mp_kernel" and info["passes"] >= 2
        a = sim.advance(70)
        b = sim.advance(80)
        snaps = [sim.membrane_snapshot(w) for w in range(3)]
    rs = RefSim(net, opt)
    ra, rb = rs.advance(70), rs.advance(80)
    assert ra.total_spikes > 0 and rb.total_spikes > 0
    assert_same(a, ra)
    assert_same(b, rb)
    for w in range(3):
        assert np.array_equal(snaps[w], rs.membrane_snapshot(w))


def test_crossing_matrix_matches_reference():
    """crossing_matrix (netgen.cpp:331-355, BuiltNetwork::crossing) counted on
    the device from the delivery tables equals the reference pipeline's, for
    loaded tables and for tables generated on the device."""
    from paper_2308_01241_b200 import netgen
    cfg = make_config(seed=13, voxels=6, npv=300, k_in=25, rho=0.3, workers=3,
                      partition="greedy")
    net = RefNet(cfg)
    ref = net.crossing()
    assert ref.sum() == net.tables.synapse_count and ref[0, 1] + ref[1, 0] > 0
    with SimInstance(net.tables, SimOptions(steps=1)) as sim:
        assert np.array_equal(sim.crossing_matrix(), ref)
    with netgen.GeneratedSimInstance(netgen.build_network(cfg), SimOptions(steps=1)) as sim:
        assert np.array_equal(sim.crossing_matrix(), ref)


def test_set_conductances_batch_equals_item_by_item():
    """vxb_set_conductances_batch = set_conductances item by item, in order:
    the later of two sets of one (unit, receptor) wins, a bad value stops the
    sequence after staging that item's valid prefix (engine.cpp:829-844)."""
    net = RefNet(hot_cfg(seed=41, voxels=3, npv=200, k_in=15, rho=0.3), even_workers=2)
    units = net.tables.units
    rng = np.random.default_rng(3)
    items = [(u, r, rng.uniform(0.5, 2.0, int(units["neurons"][u])).astype(np.float32))
             for u in range(units.shape[0]) for r in (0, 2)]
    bad = items[5][2].copy()
    bad[7] = -1.0
    seq_items = items[:5] + [(items[5][0], items[5][1], bad)] + items[6:]
    opt = SimOptions(steps=40, probe_gids=[3, 300, 599])
    with SimInstance(net.tables, opt) as a, SimInstance(net.tables, opt) as b:
        for u, r, v in items[:3] + [items[1]]:  # duplicate key: sequential path
            a.set_conductances(u, r, v)
        a.set_conductances_batch(items[:3] + [items[1]])  # no-op duplicate of the same values
        b.set_conductances_batch(items[:3] + [items[1]])
        with pytest.raises(ConfigError):
            for u, r, v in seq_items:
                a.set_conductances(u, r, v)
        with pytest.raises(ConfigError):
            b.set_conductances_batch(seq_items)
        assert b.failed_index == 5
        ra, rb = a.advance(40), b.advance(40)
        assert ra.total_spikes == rb.total_spikes > 0
        assert raster_set(ra.raster) == raster_set(rb.raster)
        assert np.array_equal(ra.rates.counts, rb.rates.counts)
        for pa, pb in zip(ra.probes, rb.probes):
            assert np.array_equal(pa.v, pb.v) and np.array_equal(pa.i_syn, pb.i_syn)
        for w in range(2):
            assert np.array_equal(a.membrane_snapshot(w), b.membrane_snapshot(w))


def test_tile_spike_staging_overflow_matches_reference(monkeypatch):
    """A synchronized burst larger than a tile's spike staging (kSpkStage =
    1024 per CTA and step): 1 500 forced spikes in the first tile at one step
    take the direct log / queue path of the SM-tile kernel; raster, rates and
    final V equal the reference's."""
    set_path(monkeypatch, "tile")
    net = RefNet(make_config(seed=5, voxels=16, npv=10000, k_in=10, steps=20))
    w0 = net.tables.workers[0]
    gids = [int(g) for g in w0.neurons["gid"][:1500]]
    opt = SimOptions(steps=20, forced_spikes=[ForcedSpike(5, g) for g in gids])
    with SimInstance(net.tables, opt) as sim:
        assert sim.schedule_info()["path"] == "sm_tile"
        assert sim.schedule_info()["tile_neurons"] > 1024
        r = sim.advance(20)
        snaps = [sim.membrane_snapshot(w) for w in range(sim.workers)]
    ref = RefSim(net, opt).advance(20)
    assert r.total_spikes == ref.total_spikes
    assert int((r.raster["step"] == 5).sum()) >= 1500
    assert raster_set(r.raster) == raster_set(ref.raster)
    rs = RefSim(net, opt)
    rs.advance(20)
    for w in range(len(snaps)):
        assert np.array_equal(snaps[w], rs.membrane_snapshot(w)), w


@pytest.mark.parametrize("path", ["tile", "l2"])
def test_divergence_reports_the_references_neuron_and_step(monkeypatch, path):
    """An infinite injection into one voxel from step 3: both paths report the
    reference's SimError text (the smallest diverging neuron of the earliest
    step) — on the SM-tile path the CTAs stop on their own, without a grid
    barrier, and must still agree on it."""
    set_path(monkeypatch, path)
    net = RefNet(quiet_cfg(seed=8, voxels=6, npv=600, k_in=4))
    # (checked against the C restatement of the reference step, which takes
    # the options as a struct: the reference's JSON options have no infinity)
    opt = SimOptions(steps=12, injections=[Injection(3, 12, 2, float("inf"))])
    with pytest.raises(SimError) as ref_err:
        OracleSim(net.tables, opt).advance(12)
    with SimInstance(net.tables, opt) as sim:
        assert sim.schedule_info()["path"] == ("sm_tile" if path == "tile" else "l2_atomic")
        with pytest.raises(SimError) as gpu_err:
            sim.advance(12)
    assert str(gpu_err.value) == str(ref_err.value)
    assert "membrane potential diverged" in str(gpu_err.value)
