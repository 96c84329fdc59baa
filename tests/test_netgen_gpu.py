"""GPU tests of on-device network generation: the worker tables sampled on
the B200 must equal emit_tables' output from the reference pipeline
(netgen.cpp:51-316) byte for byte, and a simulation over generated tables
must equal the reference engine's run on its own tables."""
import numpy as np
import pytest

from paper_2308_01241_b200 import netgen
from paper_2308_01241_b200.engine import SimOptions
from refnet import RefNet, RefSim, make_config, raster_set
from test_netgen import CFGS

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", CFGS[:5] + CFGS[6:])
def test_generated_tables_match_emit_tables(cfg):
    ref = RefNet(cfg)
    gen = netgen.generate_tables(netgen.build_network(cfg))
    assert len(gen.workers) == len(ref.tables.workers)
    for a, b in zip(gen.workers, ref.tables.workers):
        assert np.array_equal(a.row_base, b.row_base)
        assert np.array_equal(a.neurons, b.neurons), "neuron records differ"
        assert np.array_equal(a.synapses, b.synapses), "synapse rows differ"
    assert np.array_equal(gen.unit_local_base, ref.tables.unit_local_base)


def test_generated_simulation_matches_reference():
    cfg = make_config(seed=1401, voxels=100, npv=1000, k_in=100, rho=6 / 25, workers=1)
    net = netgen.build_network(cfg)
    probes = [i * 8321 + 17 for i in range(12)]
    opt = SimOptions(steps=300, probe_gids=probes)
    with netgen.GeneratedSimInstance(net, opt) as sim:
        gpu = sim.advance(300)
    ref = RefSim(RefNet(cfg), opt).advance(300)
    assert gpu.total_spikes == ref.total_spikes > 0
    assert raster_set(gpu.raster) == raster_set(ref.raster)
    assert np.array_equal(np.stack([p.v for p in gpu.probes]), ref.probe_v)
    assert np.array_equal(np.stack([p.i_syn for p in gpu.probes]), ref.probe_i)
    assert gpu.flops == ref.flops
