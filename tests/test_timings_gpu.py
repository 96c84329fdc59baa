"""StepTimings rows of the CUDA engine: wire-byte accounting and the timing
identities of the reference's acceptance criterion 9 (acceptance.cpp:651-742).

The reference counts, per (step, worker), the bytes of every spike batch it
sends and receives — encode_batch's 12-byte header plus LEB128 varints of the
ascending local ids' deltas (transport.cpp:10-55) — split by node
(worker / workers_per_node), and anchors the send/receive spans so that they
telescope (engine.cpp:495-523, 570-597).  The GPU engine hosts the workers on
one device (or one per rank) and has no sender/receiver threads, but its rows
must carry the same byte counters and satisfy the same identities.
"""
import numpy as np
import pytest

from paper_2308_01241_b200.engine import SimInstance, SimOptions
from refnet import RefNet, RefSim

pytestmark = pytest.mark.gpu


def _varint_len(v):
    n = 1
    while v >= 0x80:
        v >>= 7
        n += 1
    return n


def _encode_size(ids):  # encode_batch (transport.cpp:33-55)
    size, prev = 12, 0
    for k, x in enumerate(ids):
        size += _varint_len(x if k == 0 else x - prev)
        prev = x
    return size


def _criterion9_cfg(quiet=False):
    reg = {"k_in": 30}
    if quiet:
        reg.update(ou_mean=0.0, ou_sigma=0.0)
    return {"seed": 77, "steps": 60, "workers": 4, "workers_per_node": 2, "scheduler": "loopback",
            "connectome": {"kind": "ring", "voxels": 3, "neurons_per_voxel": 80},
            "partition": {"method": "greedy"}, "regions": {"subcortex": reg}}


@pytest.mark.parametrize("path", ["tile", "l2", "mp"])
def test_statistics_identities_criterion9(monkeypatch, path):
    monkeypatch.setenv("VXB_TUNING", "1")
    monkeypatch.setenv("VXB_PATH", "l2" if path == "l2" else "tile")
    if path == "mp":
        monkeypatch.setenv("VXB_TILE_PER", "32")
    cfg = _criterion9_cfg()
    net = RefNet(cfg)
    opt = SimOptions(steps=60, workers_per_node=2)
    with SimInstance(net.tables, opt) as sim:
        run = sim.advance(60)
    assert run.total_spikes > 0
    t = run.timings
    W = 4
    assert t.shape[0] == 60 * W
    # send / receive splits telescope; copy markers sit on their anchors
    tt = t["t"]
    assert np.array_equal(t["send_intra_ns"] + t["send_inter_ns"], tt[:, 8] - tt[:, 7])
    assert np.array_equal(t["recv_intra_ns"] + t["recv_inter_ns"], tt[:, 10] - tt[:, 9])
    assert np.array_equal(tt[:, 3], tt[:, 0]) and np.array_equal(tt[:, 4], tt[:, 0])
    assert np.array_equal(tt[:, 5], tt[:, 1]) and np.array_equal(tt[:, 6], tt[:, 1])
    # byte counters equal re-encoded payload sizes, split by node
    spikes = {}
    for e in run.raster:
        spikes.setdefault((int(e["step"]), int(e["worker"])), []).append(int(e["local"]))
    node = lambda w: w // 2  # noqa: E731
    masks = [wt.neurons["dst_mask"] for wt in net.tables.workers]
    for r in t:
        s, w = int(r["step"]), int(r["worker"])
        local = spikes.get((s, w), [])
        assert int(r["spikes"]) == len(local)
        sent = {True: 0, False: 0}
        recv = {True: 0, False: 0}
        for d in range(W):
            if d == w:
                continue
            ids = [l for l in local if (int(masks[w][l]) >> d) & 1]
            sent[node(d) == node(w)] += _encode_size(ids)
            sids = [l for l in spikes.get((s, d), []) if (int(masks[d][l]) >> w) & 1]
            recv[node(d) == node(w)] += _encode_size(sids)
        assert int(r["bytes_sent_intra"]) == sent[True] and int(r["bytes_sent_inter"]) == sent[False]
        assert int(r["bytes_recv_intra"]) == recv[True] and int(r["bytes_recv_inter"]) == recv[False]
    # ... and equal the reference engine's own rows
    rs = RefSim(net, opt)
    rs.advance(60)
    ref = rs.timings()
    for f in ("step", "worker", "spikes", "bytes_sent_intra", "bytes_sent_inter",
              "bytes_recv_intra", "bytes_recv_inter"):
        assert np.array_equal(t[f], ref[f]), f


def test_silent_network_byte_floor_and_static_flops():
    """acceptance.cpp:718-741: a silent network's spike-dependent FLOP
    counters stay zero, the static ones are exact, and every batch is an
    empty 12-byte barrier message (12 intra + 24 inter per row)."""
    cfg = _criterion9_cfg(quiet=True)
    cfg["steps"] = 50
    net = RefNet(cfg)
    with SimInstance(net.tables, SimOptions(steps=50, workers_per_node=2)) as sim:
        run = sim.advance(50)
    assert run.total_spikes == 0
    assert run.flops["gating_inner"] == 0 and run.flops["gating_outer"] == 0
    n = net.total_neurons
    assert run.flops["membrane"] == 6 * n * 50
    assert run.flops["gating_decay"] == 12 * n * 50
    assert run.flops["current"] == 16 * n * 50
    assert np.all(run.timings["bytes_sent_intra"] == 12)
    assert np.all(run.timings["bytes_sent_inter"] == 24)
    assert np.all(run.timings["bytes_recv_intra"] == 12)
    assert np.all(run.timings["bytes_recv_inter"] == 24)


def test_timings_without_raster_keep_bytes():
    """record_raster = false still yields the byte counters (the spike log is
    kept per step internally) and no raster."""
    net = RefNet(_criterion9_cfg())
    opt_r = SimOptions(steps=60, workers_per_node=2)
    opt_n = SimOptions(steps=60, workers_per_node=2, record_raster=False)
    with SimInstance(net.tables, opt_r) as a, SimInstance(net.tables, opt_n) as b:
        ra, rb = a.advance(60), b.advance(60)
    assert rb.raster.shape[0] == 0 and ra.raster.shape[0] > 0
    for f in ("bytes_sent_intra", "bytes_sent_inter", "bytes_recv_intra", "bytes_recv_inter"):
        assert np.array_equal(ra.timings[f], rb.timings[f]), f
