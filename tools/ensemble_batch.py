"""Ensemble members advanced one after another vs together
(vxb_advance_members): wall time of one assimilation window for M members of
a donor (EnsembleMember::run_window, assim.cpp:91-107).

    python tools/ensemble_batch.py [--members 8] [--voxels 100] [--steps 100] [--path l2|tile]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
ap = argparse.ArgumentParser()
ap.add_argument("--members", type=int, default=8)
ap.add_argument("--voxels", type=int, default=100)
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--path", default="")
args = ap.parse_args()
if args.path:
    os.environ["VXB_TUNING"] = "1"
    os.environ["VXB_PATH"] = args.path
import bench  # noqa: E402
from paper_2308_01241_b200 import netgen  # noqa: E402
from paper_2308_01241_b200.engine import SimOptions, advance_members  # noqa: E402

net = netgen.build_network(bench.workload_cfg(voxels=args.voxels))
opt = SimOptions(steps=args.steps, record_raster=False, record_timings=False)
with netgen.GeneratedSimInstance(net, opt) as donor:
    members = [donor.member() for _ in range(args.members)]
    path = members[0].schedule_info()["path"]
    out = {"members": args.members, "neurons": net.total_neurons, "steps": args.steps,
           "path": path}
    for rep in range(3):
        t0 = time.perf_counter()
        ev = sum(m.advance(args.steps).events for m in members)
        t1 = time.perf_counter()
        res = advance_members(members, args.steps)
        t2 = time.perf_counter()
        ev2 = sum(r.events for r in res)
    out.update(serial_s=t1 - t0, together_s=t2 - t1, serial_events=ev, together_events=ev2,
               speedup=(t1 - t0) / (t2 - t1))
    for m in members:
        m.close()
print(json.dumps(out))
