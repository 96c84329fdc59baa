"""Dry run of the per-rank device memory for a benchmark network (no GPU
needed): netgen.memory_plan over the partition bench.py would build.

    python tools/memory_plan.py [--workload config5|config3|config2] [--gpus 8]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2308_01241_b200 import netgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="config5")
ap.add_argument("--gpus", type=int, default=8)
args = ap.parse_args()
if args.workload == "config5":
    cfg = bench.config5_cfg(workers=args.gpus)
elif args.workload == "config3":
    cfg = bench.dti_cfg(workers=args.gpus)
else:
    cfg = bench.workload_cfg(voxels=100 * args.gpus, workers=args.gpus)
    cfg["partition"]["method"] = "sequential"
net = netgen.build_network(cfg)
plan = netgen.memory_plan(net)
print(json.dumps({"workload": args.workload, "gpus": args.gpus, "neurons": net.total_neurons,
                  "synapses": net.synapse_count, "ranks": plan}, indent=1))
