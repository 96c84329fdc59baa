"""Phase profile of one config-2 advance (VXB_TUNING=1 VXB_PHASE_PROFILE=1):
per-phase time and, per CTA, when each part of the step kernel ends.

    python tools/phase_profile.py [--steps 50] [--voxels 100] [--path tile|l2]
"""
import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--voxels", type=int, default=100)
ap.add_argument("--path", default="")
ap.add_argument("--silent", action="store_true", help="ou_mean = 0: no spikes")
ap.add_argument("--cons", default="", help="VXB_TILE_CONS (consumer warps)")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--workload", default="config2", choices=["config2", "config3"])
args = ap.parse_args()
os.environ["VXB_TUNING"] = "1"
if os.environ.get("VXB_PROF_DUMP") and int(os.environ.get("WORLD_SIZE", "1")) > 1:
    os.environ["VXB_PROF_DUMP"] += f".rank{os.environ.get('RANK', '0')}"
os.environ["VXB_PHASE_PROFILE"] = "1"
if args.path:
    os.environ["VXB_PATH"] = args.path
if args.cons:
    os.environ["VXB_TILE_CONS"] = args.cons
import bench  # noqa: E402
from paper_2308_01241_b200 import netgen  # noqa: E402
from paper_2308_01241_b200.engine import SimOptions  # noqa: E402

cfg = bench.workload_cfg(voxels=args.voxels) if args.workload == "config2" else bench.dti_cfg()
if args.silent:
    cfg["regions"]["subcortex"]["ou_mean"] = 0.0

ws = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
if ws > 1:  # under torchrun: config 2 weak-scaled, one rank per GPU
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    cfg = bench.workload_cfg(voxels=args.voxels * ws, workers=ws)
    cfg["partition"]["method"] = "sequential"
    if args.silent:
        cfg["regions"]["subcortex"]["ou_mean"] = 0.0
net = netgen.build_network(cfg)
opt = SimOptions(steps=args.steps, record_raster=False, record_timings=False, device=rank)
sim = (netgen.DistributedSimInstance(net, opt, rank, ws) if ws > 1
       else netgen.GeneratedSimInstance(net, opt))
if rank == 0:
    print(sim.schedule_info(), flush=True)
for _ in range(args.reps):
    r = sim.advance(args.steps)
    print(f"rank {rank}: advance {r.device_ms / args.steps * 1e3:.1f} us/step, {r.events} events, "
          f"{r.total_spikes} spikes, exchange wait {r.exchange_wait_ms / args.steps * 1e3:.1f} us/step",
          flush=True)
sim.close()
