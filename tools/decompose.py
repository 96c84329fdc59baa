"""Split the step time of the config-2 workload into neuron update vs
delivery: the same 1M-neuron network run silent (ou_mean = 0: no spikes, the
OU noise still drawn) and at its ~10 Hz operating point."""
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
    base = bench.workload_cfg()
    quiet = json.loads(json.dumps(base))
    quiet["regions"]["subcortex"]["ou_mean"] = 0.0
    print(json.dumps({"silent": run(quiet), "10hz": run(base)}), flush=True)
