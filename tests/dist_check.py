"""Multi-GPU parity check, run under torchrun (one process per GPU):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/dist_check.py [cfg-json]

Every rank runs its worker of an N-worker partition on its own GPU with the
NVLink spike exchange; rank 0 gathers the raster, rates, probes and final
membrane state and compares them with the reference engine (oracle/_ref) on
the same network and partition, bit for bit.  Prints one JSON line.
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2308_01241_b200 import netgen  # noqa: E402
from paper_2308_01241_b200.engine import HemoParams, SimOptions  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    cfg = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {
        "seed": 1401, "dt_ms": 1.0, "steps": 300, "workers": world,
        "connectome": {"kind": "ring", "voxels": 12, "neurons_per_voxel": 2000},
        "partition": {"method": "greedy"},
        "regions": {"subcortex": {"k_in": 100, "ou_mean": 300.0}}}
    cfg["workers"] = world
    steps = cfg["steps"]
    net = netgen.build_network(cfg)
    probes = [17, 5000, net.total_neurons - 1]
    opt = SimOptions(steps=steps, dt_ms=cfg["dt_ms"], probe_gids=probes, device=local)
    sim = netgen.DistributedSimInstance(net, opt, rank, world)
    # BOLD readout across ranks: voxel counts summed, hemodynamics on the totals
    sim.set_hemodynamics(HemoParams(), baseline_hz=10.0, sample_every=50)
    r1 = sim.advance(steps // 3)
    r2 = sim.advance(steps - steps // 3)
    snap = sim.membrane_snapshot(rank)
    w_gids = None
    mine = {
        "raster": sorted(zip(r1.raster["step"].tolist() + r2.raster["step"].tolist(),
                             r1.raster["gid"].tolist() + r2.raster["gid"].tolist())),
        "rates": np.concatenate([r1.rates.counts, r2.rates.counts], axis=1),
        "pv": np.concatenate([np.stack([p.v for p in r.probes]) for r in (r1, r2)], axis=1),
        "pi": np.concatenate([np.stack([p.i_syn for p in r.probes]) for r in (r1, r2)], axis=1),
        "flops": {k: r1.flops[k] + r2.flops[k] for k in r1.flops},
        "snap": snap,
        "bold": [r1.bold, r2.bold],
        # this rank's StepTimings rows (its own worker's rows are filled)
        "timings": [r.timings[r.timings["worker"] == rank] for r in (r1, r2)],
    }
    crossing = sim.crossing_matrix()  # collective
    out = [None] * world
    dist.all_gather_object(out, mine)
    sim.close()
    if rank == 0:
        from refnet import RefNet, RefSim
        ref_net = RefNet(cfg)
        crossing_ok = bool(np.array_equal(crossing, ref_net.crossing()))
        rs = RefSim(ref_net, SimOptions(steps=steps, dt_ms=cfg["dt_ms"], probe_gids=probes))
        a = rs.advance(steps // 3)
        ta = rs.timings()
        b = rs.advance(steps - steps // 3)
        tb = rs.timings()
        ref_raster = sorted(zip(a.raster["step"].tolist() + b.raster["step"].tolist(),
                                a.raster["gid"].tolist() + b.raster["gid"].tolist()))
        raster = sorted(x for o in out for x in o["raster"])
        rates = sum(o["rates"] for o in out)
        # a probe is recorded by the rank that owns its neuron (zeros elsewhere)
        pv = sum(o["pv"] for o in out)
        pi = sum(o["pi"] for o in out)
        ref_pv = np.concatenate([a.probe_v, b.probe_v], axis=1)
        ref_pi = np.concatenate([a.probe_i, b.probe_i], axis=1)
        fl = {k: sum(o["flops"][k] for o in out) for k in out[0]["flops"]}
        ref_fl = {k: a.flops[k] + b.flops[k] for k in a.flops}
        snaps_ok = all(np.array_equal(out[w]["snap"], rs.membrane_snapshot(w)) for w in range(world))
        # window_bold (assim.cpp:51-71) on the reference engine's rates
        from refnet import ref_window_bold
        units = net.arrays["units"]
        vox_n = np.zeros(len(net.layout.voxels), np.uint64)
        np.add.at(vox_n, units["voxel"].astype(np.int64), units["neurons"].astype(np.uint64))
        st = np.tile([0.0, 1.0, 1.0, 1.0], (len(vox_n), 1))
        ref_bold = [ref_window_bold(HemoParams(), x.rates, units["voxel"], vox_n,
                                    cfg["dt_ms"] * 1e-3, 10.0, 50, st) for x in (a, b)]
        bold_ok = all(np.array_equal(o["bold"][k], out[0]["bold"][k])
                      for o in out for k in range(2))  # every rank holds the same series
        for k in range(2):
            g, r = out[0]["bold"][k], ref_bold[k]
            bold_ok = bold_ok and g.shape == r.shape and \
                float(np.max(np.abs(g - r))) <= 1e-12 * float(np.max(np.abs(r))) + 1e-15
        # wire-byte counters (engine.cpp:495-523): every row equals the
        # reference's; send / receive spans telescope
        timings_ok = True
        for k, tref in enumerate((ta, tb)):
            rows = np.concatenate([o["timings"][k] for o in out])
            rows = rows[np.lexsort((rows["worker"], rows["step"]))]
            timings_ok = timings_ok and rows.shape == tref.shape
            for f in ("step", "worker", "spikes", "bytes_sent_intra", "bytes_sent_inter",
                      "bytes_recv_intra", "bytes_recv_inter"):
                timings_ok = timings_ok and bool(np.array_equal(rows[f], tref[f]))
            tt = rows["t"]
            timings_ok = timings_ok and bool(np.array_equal(
                rows["recv_intra_ns"] + rows["recv_inter_ns"], tt[:, 10] - tt[:, 9]))
            timings_ok = timings_ok and bool(np.array_equal(
                rows["send_intra_ns"] + rows["send_inter_ns"], tt[:, 8] - tt[:, 7]))
        res = {
            "world": world, "spikes": len(raster), "ref_spikes": len(ref_raster),
            "timings_equal": timings_ok, "crossing_equal": crossing_ok,
            "bold_equal": bool(bold_ok),
            "raster_equal": raster == ref_raster,
            "rates_equal": bool(np.array_equal(rates, np.concatenate([a.rates, b.rates], axis=1))),
            "probe_v_equal": bool(np.array_equal(pv, ref_pv)),
            "probe_i_equal": bool(np.array_equal(pi, ref_pi)),
            "flops_equal": fl == ref_fl, "snapshots_equal": snaps_ok,
            "gating_outer": fl["gating_outer"],
        }
        res["pass"] = all(v for k, v in res.items() if k.endswith("_equal")) and res["spikes"] > 0
        print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main_full():
    """Full-size property (BASELINE config 2 weak-scaling network, 1M neurons
    per GPU, K = 1000): the N-GPU run with the NVLink exchange equals the same
    N-worker network hosted on one GPU (raster, rates, state)."""
    import bench
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    steps = 40
    cfg = bench.workload_cfg(voxels=100 * world, workers=world)
    cfg["partition"] = {"method": "sequential"}
    net = netgen.build_network(cfg)
    opt = SimOptions(steps=steps, record_raster=True, record_timings=False, device=local)
    sim = netgen.DistributedSimInstance(net, opt, rank, world)
    r = sim.advance(steps)
    mine = {"raster": np.stack([r.raster["step"].astype(np.int64), r.raster["gid"].astype(np.int64)], 1),
            "rates": r.rates.counts, "snap": sim.membrane_snapshot(rank), "events": r.events}
    sim.close()
    out = [None] * world
    dist.all_gather_object(out, mine)
    if rank == 0:
        raster = np.concatenate([o["raster"] for o in out])
        raster = raster[np.lexsort((raster[:, 1], raster[:, 0]))]
        with netgen.GeneratedSimInstance(net, SimOptions(steps=steps, record_raster=True,
                                                         record_timings=False, device=local)) as one:
            q = one.advance(steps)
            snaps = [one.membrane_snapshot(w) for w in range(world)]
        qr = np.stack([q.raster["step"].astype(np.int64), q.raster["gid"].astype(np.int64)], 1)
        qr = qr[np.lexsort((qr[:, 1], qr[:, 0]))]
        res = {"world": world, "mode": "full", "spikes": int(raster.shape[0]),
               "events": int(sum(o["events"] for o in out)), "one_gpu_events": int(q.events),
               "raster_equal": bool(raster.shape == qr.shape and np.array_equal(raster, qr)),
               "rates_equal": bool(np.array_equal(sum(o["rates"] for o in out), q.rates.counts)),
               "snapshots_equal": all(np.array_equal(out[w]["snap"], snaps[w]) for w in range(world))}
        res["pass"] = all(v for k, v in res.items() if k.endswith("_equal")) and res["spikes"] > 0
        print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main_abort():
    """Cross-rank abort (engine.cpp:117-142, 483-484): the last rank's
    neurons diverge (an infinite injection current drives V to inf at step 30);
    that rank reports the divergence and every other rank must leave its step
    barrier with "simulation aborted while waiting on the step barrier" at
    once, not after recv_timeout_ms (30 s)."""
    import time
    from paper_2308_01241_b200.engine import Injection, SimError
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    cfg = {"seed": 1401, "dt_ms": 1.0, "steps": 200, "workers": world,
           "connectome": {"kind": "ring", "voxels": 12, "neurons_per_voxel": 2000},
           "partition": {"method": "sequential"},
           "regions": {"subcortex": {"k_in": 100, "ou_mean": 300.0}}}
    net = netgen.build_network(cfg)
    last_voxel = len(net.layout.voxels) - 1  # sequential partition: on rank world - 1
    opt = SimOptions(steps=200, device=local, recv_timeout_ms=30000,
                     injections=[Injection(30, 200, last_voxel, float("inf"))])
    sim = netgen.DistributedSimInstance(net, opt, rank, world)
    t0 = time.perf_counter()
    msg = ""
    try:
        sim.advance(200)
    except SimError as e:
        msg = str(e)
    dt = time.perf_counter() - t0
    # a failed instance rejects further advances (engine.cpp:765-766)
    try:
        sim.advance(1)
        rejected = False
    except SimError:
        rejected = True
    out = [None] * world
    dist.all_gather_object(out, {"rank": rank, "msg": msg, "seconds": dt, "rejected": rejected})
    if rank == 0:
        div = out[world - 1]["msg"].startswith("membrane potential diverged")
        others = all(o["msg"] == "simulation aborted while waiting on the step barrier"
                     for o in out[:world - 1])
        fast = max(o["seconds"] for o in out) < 5.0
        res = {"world": world, "mode": "abort", "ranks": out, "diverged_equal": div,
               "aborted_equal": others, "fast_equal": fast,
               "rejected_equal": all(o["rejected"] for o in out)}
        res["pass"] = div and others and fast and res["rejected_equal"]
        print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--full":
        main_full()
    elif len(sys.argv) > 1 and sys.argv[1] == "--abort":
        main_abort()
    else:
        main()
