"""VXTB v1 table files (netgen.cpp:359-539): byte compatibility with the
reference's writer and reader in both directions, integrity checks, and the
engine running from loaded tables."""
import json

import numpy as np
import pytest

from paper_2308_01241_b200 import netgen, tables_io
from paper_2308_01241_b200.engine import SimError, SimOptions
from refnet import RefNet, RefSim, make_config, raster_set

CFG = make_config(seed=8, voxels=5, npv=120, k_in=12, rho=0.3, workers=3, partition="greedy")


def _same_tables(a, b):
    assert len(a.workers) == len(b.workers)
    for x, y in zip(a.workers, b.workers):
        assert (x.worker, x.worker_count, x.seed) == (y.worker, y.worker_count, y.seed)
        assert np.array_equal(x.neurons, y.neurons)
        assert np.array_equal(x.synapses, y.synapses)
        assert np.array_equal(x.row_base, y.row_base)
    assert np.array_equal(a.unit_worker, b.unit_worker)
    assert np.array_equal(a.unit_local_base, b.unit_local_base)


def test_fnv1a_known_answers():
    assert tables_io.fnv1a(b"") == 0xCBF29CE484222325
    assert tables_io.fnv1a(b"a") == 0xAF63DC4C8601EC8C
    assert tables_io.fnv1a(b"foobar") == 0x85944171F73967E8


def test_load_reference_written_tables(tmp_path):
    ref = RefNet(CFG)
    ref.save_tables(tmp_path)
    b = netgen.build_network(CFG)
    t = tables_io.load_tables(tmp_path, b.arrays["units"], len(b.layout.voxels))
    _same_tables(t, ref.tables)


def test_reference_loads_our_tables(tmp_path):
    ref = RefNet(CFG)
    tables_io.save_tables(ref.tables, tmp_path)
    # byte-identical to the reference's own files and manifest hashes
    ref.save_tables(tmp_path / "ref")
    for w in range(3):
        name = f"worker_{w:03d}.bin"
        assert (tmp_path / name).read_bytes() == (tmp_path / "ref" / name).read_bytes()
    back = RefNet(CFG, tables_dir=tmp_path)
    _same_tables(back.tables, ref.tables)


def test_integrity_errors(tmp_path):
    ref = RefNet(CFG)
    tables_io.save_tables(ref.tables, tmp_path)
    b = netgen.build_network(CFG)
    units, nv = b.arrays["units"], len(b.layout.voxels)
    f = tmp_path / "worker_001.bin"
    raw = bytearray(f.read_bytes())
    raw[100] ^= 0xFF
    f.write_bytes(bytes(raw))
    with pytest.raises(SimError, match="table hash mismatch"):
        tables_io.load_tables(tmp_path, units, nv)
    f.write_bytes(bytes(raw[:-5]))
    m = json.loads((tmp_path / "manifest.json").read_text())
    m["files"][1]["fnv1a"] = f"{tables_io.fnv1a(f.read_bytes()):016x}"
    (tmp_path / "manifest.json").write_text(json.dumps(m))
    with pytest.raises(SimError, match="truncated table file"):
        tables_io.load_tables(tmp_path, units, nv)
    with pytest.raises(SimError, match="not a worker table file"):
        g = tmp_path / "bad.bin"
        g.write_bytes(b"\0" * 64)
        tables_io.load_worker_table(g)


@pytest.mark.gpu
def test_engine_runs_from_table_files(tmp_path):
    from paper_2308_01241_b200.engine import SimInstance
    ref = RefNet(CFG)
    ref.save_tables(tmp_path)
    b = netgen.build_network(CFG)
    t = tables_io.load_tables(tmp_path, b.arrays["units"], len(b.layout.voxels))
    opt = SimOptions(steps=100, probe_gids=[3, 300])
    with SimInstance(t, opt) as sim:
        g = sim.advance(100)
    r = RefSim(ref, opt).advance(100)
    assert g.total_spikes == r.total_spikes > 0
    assert raster_set(g.raster) == raster_set(r.raster)
    assert np.array_equal(np.stack([p.v for p in g.probes]), r.probe_v)
