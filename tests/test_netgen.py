"""CPU tests of the host half of network generation (paper_2308_01241_b200/
netgen.py): config parsing, connectome generators, layout and partitioners
must reproduce the reference pipeline (pipeline.cpp:49-125) exactly."""
import numpy as np
import pytest

from paper_2308_01241_b200 import netgen
from paper_2308_01241_b200.engine import ConfigError
from refnet import RefNet, make_config

CFGS = [
    make_config(seed=5, voxels=3, npv=60, k_in=8, rho=0.4, workers=3, partition="greedy"),
    make_config(seed=11, voxels=20, npv=300, k_in=40, rho=0.3, workers=4, partition="greedy",
                kind="uniform", connectome={"sparsity": 0.1}),
    make_config(seed=12, voxels=12, npv=103, k_in=20, rho=0.5, workers=3,
                partition="sequential", kind="two_block", connectome={"scramble": True}),
    make_config(seed=13, voxels=5, npv=97, k_in=12, rho=0.2, workers=3, partition="exact"),
    make_config(seed=14, voxels=1, npv=1234, k_in=50, workers=1),
    make_config(seed=1401, voxels=100, npv=1000, k_in=100, rho=6 / 25, workers=8,
                partition="greedy"),
    make_config(seed=3, voxels=40, npv=500, k_in=30, rho=0.3, workers=8, partition="greedy",
                kind="uniform", connectome={"sparsity": 0.0072, "gm_sigma": 0.5},
                extra_region={"ou_mean": 250.0, "weight_spread": [0.3, 0.1, 0.2, 0.2],
                              "dual_receptor": False, "split_ratio": 0.3}),
]


@pytest.mark.parametrize("cfg", CFGS)
def test_layout_and_partition_match_reference(cfg):
    ref = RefNet(cfg)
    b = netgen.build_network(cfg)
    t = ref.tables
    assert np.array_equal(t.units, b.arrays["units"])
    assert np.array_equal(t.unit_worker, b.arrays["unit_worker"])
    assert b.synapse_count == t.synapse_count
    assert b.total_neurons == ref.total_neurons


def test_partition_objective_prefers_greedy():
    cfg = make_config(seed=2, voxels=24, npv=200, k_in=30, rho=0.4, workers=4)
    g = netgen.build_network(cfg, method="greedy")
    s = netgen.build_network(cfg, method="sequential")
    fg = netgen.partition_objective(g.unit_graph, g.unit_worker, 4)
    fs = netgen.partition_objective(s.unit_graph, s.unit_worker, 4)
    assert fg <= fs


def test_connectome_text_round_trip():
    cfg = netgen.parse_config(make_config(seed=3, voxels=30, npv=10, kind="uniform",
                                          connectome={"sparsity": 0.05, "gm_sigma": 0.4}))
    g = netgen.build_connectome(cfg)
    h = netgen.load_connectome_text(netgen.save_connectome_text(g))
    assert h.edges == g.edges and h.neuron_count == g.neuron_count
    assert h.gm_weight == g.gm_weight and h.region == g.region


def test_config_validation():
    with pytest.raises(ConfigError, match="unknown key"):
        netgen.parse_config({"seed": 1, "bogus": 2})
    with pytest.raises(ConfigError, match="unknown key"):
        netgen.parse_config({"connectome": {"kind": "ring", "nope": 1}})
    with pytest.raises(ConfigError, match="unknown partition method"):
        netgen.parse_config({"partition": {"method": "magic"}})
    with pytest.raises(ConfigError, match="ring connectome needs"):
        netgen.build_network(make_config(voxels=2, npv=10, kind="ring"))
    with pytest.raises(ConfigError, match="fewer units than workers"):
        netgen.build_network(make_config(voxels=3, npv=10, k_in=2, workers=7,
                                         partition="greedy"))
    with pytest.raises(ConfigError):
        netgen.build_network(make_config(voxels=3, npv=10, k_in=2,
                                         extra_region={"rho": 1.5}))


def test_rng_mirror_matches_reference():
    from refnet import ref_lib
    R = ref_lib()
    for a, b in [(0, 0), (5, 17), (2**63 + 1, 99)]:
        assert netgen.mix_key(a, b) == R.ref_mix_key2(a, b)
        assert netgen.stream_normal(a, b) == R.ref_stream_normal(a, b)
        assert netgen.stream_below(a, b, 13) == R.ref_stream_below(a, b, 13)


def test_llround_matches_cpp():
    for x in (0.5, 1.5, 2.4999999999999996, 2.5, 1e6 + 0.5, 0.49999999999999994, 7.0):
        assert netgen.llround(x) == int(np.floor(x + 0.5)) or x == 0.49999999999999994
    assert netgen.llround(0.49999999999999994) == 0
    assert netgen.llround(2.5) == 3 and netgen.llround(-2.5) == -3


def test_b200_byte_model_partitions_under_budget():
    cfg = make_config(seed=2, voxels=40, npv=2000, k_in=200, rho=0.3, workers=4)
    cfg["partition"] = {"method": "greedy", "byte_model": "b200"}
    b = netgen.build_network(cfg)
    loads = netgen.hbm_bytes_per_worker(b)
    assert max(loads) <= 1.1 * sum(loads) / 4  # per-GPU share cap of the b200 model
    cfg["partition"]["gamma"] = 0.5 * max(loads)
    with pytest.raises(ConfigError):
        netgen.build_network(cfg)
    with pytest.raises(ConfigError, match="byte_model"):
        netgen.parse_config({"partition": {"byte_model": "tpu"}})


def test_sample_conductances_matches_reference_tables():
    """netgen.cpp:260-261: the tables' initial per-neuron conductances are
    sample_conductances(seed, 0, unit, receptor, g_location, g_scale, n)."""
    cfg = make_config(seed=21, voxels=3, npv=200, k_in=5, rho=0.3, workers=2)
    ref = RefNet(cfg)
    b = netgen.build_network(cfg)
    g_ref = np.concatenate([w.neurons for w in ref.tables.workers])
    g_ref = g_ref[np.argsort(g_ref["gid"], kind="stable")]
    flips = 0
    for u, unit in enumerate(b.layout.units):
        pop = b.layout.pop_of_unit(u)
        rows = g_ref[unit.gid_base:unit.gid_base + unit.neurons]
        for r in range(4):
            got = netgen.sample_conductances(cfg["seed"], 0, u, r, pop.g_location[r],
                                             pop.g_scale[r], unit.neurons)
            want = rows["g"][:, r]
            assert np.allclose(got, want, rtol=2e-7, atol=0)
            flips += int((got != want).sum())
    assert flips <= 2  # numpy log/cos/exp vs glibc: rare last-ulp float flips


def test_config5_memory_plan_fits_eight_b200():
    """the whole-box network — 2e8 neurons x K = 500 =
    1e11 synapses over 8 ranks — fits each rank's 180 GB with the tables,
    offsets, L2-block offsets, exchange slots and the load-time row-sort
    scratch (netgen.memory_plan mirrors the engine's allocations)."""
    import bench
    net = netgen.build_network(bench.config5_cfg(workers=8))
    assert net.total_neurons == 200_000_000 and net.synapse_count == 100_000_000_000
    plan = netgen.memory_plan(net)
    assert len(plan) == 8
    for r in plan:
        assert r["fits"], r
        assert r["path"] == "l2_atomic" and r["l2_blocks"] >= 5
        assert 145e9 < r["buffers"]["synapse_table"] < 155e9
    # one rank per GPU at 25M neurons is near the limit: 16 ranks would halve it
    assert max(r["peak_bytes"] for r in plan) > 0.85 * plan[0]["budget_bytes"]


def test_time_model_partition_balances_step_time(tmp_path):
    """byte_model "b200_time" (per-neuron + per-event step time) balances
    the ranks' estimated step time where in-degrees differ across regions;
    the byte model balances bytes instead (multi-GPU at scale)."""
    g = netgen.make_ring(12, 2000)
    g.region = ["subcortex" if v % 3 else "brainstem" for v in range(12)]
    g.neuron_count = [2000 if v % 3 else 6000 for v in range(12)]
    path = tmp_path / "mixed.txt"
    netgen.write_connectome_file(g, path)

    def est_time(net, W):
        t = [0.0] * W
        n_fs, e_fs = netgen.TIME_MODEL_FS
        for u, x in enumerate(net.layout.units):
            k = net.layout.voxels[x.voxel].k_in
            t[net.unit_worker[u]] += x.neurons * (n_fs + e_fs * k * 10.0 * 1e-3)
        return t

    out = {}
    for bm in ("b200", "b200_time"):
        cfg = {"seed": 3, "workers": 3, "connectome": {"kind": "file", "path": str(path)},
               "partition": {"method": "greedy", "byte_model": bm, "rate_hz": 10.0},
               "regions": {"subcortex": {"k_in": 400}, "brainstem": {"k_in": 20}}}
        net = netgen.build_network(cfg)
        t = est_time(net, 3)
        out[bm] = max(t) / (sum(t) / 3)
    assert out["b200_time"] <= out["b200"] + 1e-9
