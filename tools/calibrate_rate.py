"""Rate calibration for the benchmark networks.

The default parameters at K=1000 are bistable; this sweeps g_location[AMPA]
(and optionally ou_mean) on the GPU engine and prints the mean rate of each
point so a ~10 Hz operating point can be fixed in bench.py.

    python tools/calibrate_rate.py --voxels 100 --npv 10000 --steps 500
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2308_01241_b200 import netgen  # noqa: E402
from paper_2308_01241_b200.engine import SimOptions  # noqa: E402

G_LOC = [-1.65, -4.1997, -0.2231, -2.9957]  # SURVEY.md section 6 starting point


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--voxels", type=int, default=100)
    ap.add_argument("--npv", type=int, default=10000)
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--dt", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=2)
    ap.add_argument("--ampa", type=float, nargs="+", default=[-1.8, -1.75, -1.7, -1.65, -1.6])
    ap.add_argument("--ou-mean", type=float, nargs="+", default=[None])
    a = ap.parse_args()
    for ampa, ou in [(x, y) for y in a.ou_mean for x in a.ampa]:
        reg = {"k_in": a.k, "g_location": [ampa] + G_LOC[1:]}
        if ou is not None:
            reg["ou_mean"] = ou
        cfg = {"seed": a.seed, "dt_ms": a.dt, "steps": a.steps, "workers": 1,
               "connectome": {"kind": "ring", "voxels": a.voxels, "neurons_per_voxel": a.npv},
               "partition": {"method": "sequential"}, "regions": {"subcortex": reg}}
        t0 = time.time()
        net = netgen.build_network(cfg)
        t1 = time.time()
        with netgen.GeneratedSimInstance(net, SimOptions(steps=a.steps, dt_ms=a.dt,
                                                         record_raster=False,
                                                         record_timings=False)) as sim:
            t2 = time.time()
            r = sim.advance(a.steps)
        half = r.rates.network_mean_hz(a.steps // 2)
        print(json.dumps({"ampa": ampa, "ou_mean": ou, "rate_hz": r.rates.network_mean_hz(0),
                          "rate_hz_2nd_half": half, "events": r.events,
                          "device_ms": r.device_ms, "host_build_s": t1 - t0,
                          "gen_s": t2 - t1, "synapses": net.synapse_count}), flush=True)


if __name__ == "__main__":
    main()
