"""Split the step time of a bench workload into neuron update vs delivery:
the same network run silent (ou_mean = 0: no spikes, the OU noise still
drawn) and at its ~10 Hz operating point.

    python tools/decompose.py [config2|config3] [--steps S] [--reps R] [--only silent|10hz]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2308_01241_b200 import netgen  # noqa: E402
from paper_2308_01241_b200.engine import SimOptions  # noqa: E402


def run(cfg, steps=100, reps=5):
    net = netgen.build_network(cfg)
    opt = SimOptions(steps=steps, record_raster=False, record_timings=False)
    with netgen.GeneratedSimInstance(net, opt) as sim:
        sim.advance(steps)
        ms = ev = sp = 0
        for _ in range(reps):
            r = sim.advance(steps)
            ms += r.device_ms
            ev += r.events
            sp += r.total_spikes
    return {"us_per_step": 1e3 * ms / (steps * reps), "events_per_step": ev / (steps * reps),
            "spikes_per_step": sp / (steps * reps)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="config2")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    base = bench.workload_cfg() if args.workload == "config2" else bench.dti_cfg()
    quiet = json.loads(json.dumps(base))
    quiet["regions"]["subcortex"]["ou_mean"] = 0.0
    out = {}
    if args.only in (None, "silent"):
        out["silent"] = run(quiet, args.steps, args.reps)
    if args.only in (None, "10hz"):
        out["10hz"] = run(base, args.steps, args.reps)
    print(json.dumps(out), flush=True)
