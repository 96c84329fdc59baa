"""Ensemble members on one GPU (EnsembleMember, assim.cpp:74-107): member
engines view the donor's synapse tables instead of building their own, and
must behave exactly like independent instances — and like the reference —
given the same per-member conductances."""
import numpy as np
import pytest

from paper_2308_01241_b200 import netgen
from paper_2308_01241_b200.engine import ConfigError, HemoParams, SimInstance, SimOptions
from refnet import RefNet, RefSim, make_config, raster_set

pytestmark = pytest.mark.gpu


def member_conductances(units, member):
    """assim.cpp:94-103: per-window AMPA scales of every unit, salt per member."""
    out = []
    salt = netgen.mix_key(member + 1, 1)
    for u, unit in enumerate(units):
        if unit["neurons"]:
            out.append((u, netgen.sample_conductances(7, salt, u, 0, -0.3, 0.2,
                                                      int(unit["neurons"]))))
    return out


def run(sim, conds, steps):
    for u, v in conds:
        sim.set_conductances(u, 0, v)
    r = sim.advance(steps)
    return r, [sim.membrane_snapshot(w) for w in range(sim.workers)]


def same(a, b):
    ra, sa = a
    rb, sb = b
    assert ra.total_spikes == rb.total_spikes > 0
    assert raster_set(ra.raster) == raster_set(rb.raster)
    assert np.array_equal(ra.rates.counts, rb.rates.counts)
    assert ra.flops == rb.flops
    assert all(np.array_equal(x, y) for x, y in zip(sa, sb))


def test_members_equal_independent_instances_and_reference():
    net = RefNet(make_config(seed=7, voxels=3, npv=200, k_in=20, rho=0.3, ou_mean=400.0,
                             ou_sigma=150.0), even_workers=2)
    opt = SimOptions(steps=300, dt_ms=1.0)
    units = net.tables.units
    with SimInstance(net.tables, opt) as donor:
        members = [donor.member() for _ in range(3)]
        for k, m in enumerate(members):
            conds = member_conductances(units, k)
            got = run(m, conds, 300)
            with SimInstance(net.tables, opt) as solo:
                same(got, run(solo, conds, 300))
            if k == 0:  # the reference engine with the same conductances
                rs = RefSim(net, opt)
                for u, v in conds:
                    rs.set_conductances(u, 0, v)
                ref = rs.advance(300)
                assert raster_set(got[0].raster) == raster_set(ref.raster)
                assert np.array_equal(got[0].rates.counts, ref.rates)
        # the donor itself is untouched by its members' runs
        with SimInstance(net.tables, opt) as solo:
            same(run(donor, [], 300), run(solo, [], 300))
        # members carry their own BOLD state
        members[1].set_hemodynamics(HemoParams(), baseline_hz=10.0, sample_every=50)
        r = members[1].advance(100)
        assert r.bold.shape == (2, net.tables.n_voxels) and members[2].advance(10).bold is None
        for m in members:
            m.close()


def test_generated_members_share_the_tables():
    import torch
    cfg = {"seed": 5, "dt_ms": 1.0, "connectome": {"kind": "ring", "voxels": 8,
                                                    "neurons_per_voxel": 25000},
           "regions": {"subcortex": {"k_in": 500, "ou_mean": 300.0}}}
    net = netgen.build_network(cfg)  # 2e5 neurons x 500 = 1e8 synapses = 1.2 GB of tables
    opt = SimOptions(steps=50, record_raster=True)
    with netgen.GeneratedSimInstance(net, opt) as donor:
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        m = donor.member()
        free1 = torch.cuda.mem_get_info()[0]
        assert free0 - free1 < 0.25 * 12 * net.synapse_count  # no table copy
        conds = member_conductances(net.arrays["units"], 1)
        got = run(m, conds, 50)
        m.close()
    with netgen.GeneratedSimInstance(net, opt) as solo:
        same(got, run(solo, conds, 50))


def test_member_of_a_different_network_is_rejected():
    a = RefNet(make_config(seed=3, voxels=3, npv=50, k_in=5))
    b = RefNet(make_config(seed=3, voxels=3, npv=60, k_in=5))
    with SimInstance(a.tables, SimOptions(steps=10)) as donor:
        donor._tables = b.tables  # a caller handing the wrong network
        with pytest.raises(ConfigError, match="does not match"):
            donor.member()


@pytest.mark.parametrize("path", ["l2", "tile"])
def test_members_advanced_together_equal_independent_instances(monkeypatch, path):
    """vxb_advance_members: 4 members of one donor advanced together (l2
    path: concurrently on shares of the SMs; tile path: one after another)
    over two windows, each with its own conductances, equal independent
    instances run one by one."""
    from paper_2308_01241_b200.engine import advance_members
    monkeypatch.setenv("VXB_TUNING", "1")
    monkeypatch.setenv("VXB_PATH", path)
    net = RefNet(make_config(seed=7, voxels=4, npv=500, k_in=30, rho=0.3, ou_mean=400.0,
                             ou_sigma=150.0), even_workers=2)
    opt = SimOptions(steps=200, dt_ms=1.0)
    units = net.tables.units
    with SimInstance(net.tables, opt) as donor:
        members = [donor.member() for _ in range(4)]
        together = []
        for window in range(2):
            for k, m in enumerate(members):
                for u, v in member_conductances(units, 10 * window + k):
                    m.set_conductances(u, 0, v)
            res = advance_members(members, 100)
            together.append([(r, [m.membrane_snapshot(w) for w in range(2)])
                             for r, m in zip(res, members)])
        for k in range(4):
            with SimInstance(net.tables, opt) as solo:
                for window in range(2):
                    same(together[window][k],
                         run(solo, member_conductances(units, 10 * window + k), 100))
        for m in members:
            m.close()
