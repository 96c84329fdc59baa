"""Multi-process tests of the one-process-per-GPU path.

* CPU (gloo, world size 2): the host-side exchange plumbing (destination-mask
  all-to-all) and the worker-per-rank partition.
* GPU (>= 2 devices): tests/dist_check.py under torchrun — NVLink spike
  exchange, results bit-identical to the reference engine with the same
  partition."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, store_file, q):
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    from paper_2308_01241_b200 import netgen
    # file rendezvous: no port to race for with other tests' launchers
    dist.init_process_group("gloo", init_method=f"file://{store_file}", rank=rank, world_size=world)

    def ag(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out
    # bitmap rank r builds over shard h: byte pattern (r, h)
    mine = [bytes([rank * 16 + h]) * (3 + h) for h in range(world)]
    got = netgen.exchange_masks(mine, rank, world, ag)
    ok = all(got[h] == bytes([h * 16 + rank]) * (3 + rank) for h in got) and rank not in got
    cfg = {"seed": 3, "connectome": {"kind": "ring", "voxels": 6, "neurons_per_voxel": 50},
           "regions": {"subcortex": {"k_in": 10}}}
    net = netgen.build_network(cfg, workers=world)
    ok = ok and net.workers == world and sorted(set(net.unit_worker)) == list(range(world))
    q.put((rank, ok))
    dist.destroy_process_group()


def test_mask_exchange_gloo_world2(tmp_path):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    store = tmp_path / "gloo_store"
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, str(store), q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world,env", [(2, {}), (4, {}), (2, {"VXB_TUNING": "1", "VXB_EARLY_PUBLISH": "1"}),
                                       (2, {"VXB_TUNING": "1", "VXB_DYN": "0"}),
                                       # L2-blocked delivery with peers: 4 blocks (dynamic
                                       # deal) and 2 blocks (static deal)
                                       (2, {"VXB_TUNING": "1", "VXB_PATH": "l2", "VXB_BLOCK_NEURONS": "3000"}),
                                       (2, {"VXB_TUNING": "1", "VXB_PATH": "l2", "VXB_BLOCK_NEURONS": "6000"}),
                                       (2, {"VXB_TUNING": "1", "VXB_PATH": "tile"}),
                                       (4, {"VXB_TUNING": "1", "VXB_PATH": "tile"}),
                                       # several tiles per SM is single-GPU only: with peers the
                                       # engine takes the l2 path
                                       (2, {"VXB_TUNING": "1", "VXB_PATH": "tile", "VXB_TILE_PER": "128"})])
def test_nvlink_exchange_matches_reference(world, env):
    """Default schedule, plus the optional early batch publication (4-slot
    ring), the static delivery deal and the SM-tile path (peers' batches
    scanned per tile)."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(ROOT / "tests" / "dist_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, **env})
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert lines, out.stdout + out.stderr
    res = json.loads(lines[-1])
    assert res["pass"], res
    assert res["gating_outer"] > 0  # spikes really crossed GPUs


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_fullsize_config2_two_gpus_equal_one_gpu():
    """BASELINE config 2 at full size per GPU (2 x 1M neurons, 2e9 synapses):
    the 2-GPU NVLink run equals the same 2-worker network on one GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node=2", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(ROOT / "tests" / "dist_check.py"), "--full"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert lines, out.stdout + out.stderr
    res = json.loads(lines[-1])
    assert res["pass"], res
    assert res["events"] == res["one_gpu_events"]


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("path", ["default", "tile"])
def test_divergence_on_one_rank_aborts_all_ranks(path):
    """A divergence on one rank ends every rank's advance within one step:
    the diverging rank reports it, the others the reference's "simulation
    aborted while waiting on the step barrier" (engine.cpp:483-484), well
    before the 30 s receive timeout — on the default path and on the SM-tile
    path (CTA-local stop, no grid barrier)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node=2", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(ROOT / "tests" / "dist_check.py"), "--abort"]
    env = dict(os.environ)
    if path == "tile":
        env.update(VXB_TUNING="1", VXB_PATH="tile")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert lines, out.stdout + out.stderr
    res = json.loads(lines[-1])
    assert res["pass"], res
