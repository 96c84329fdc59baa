"""Ensemble members of config 2 on one B200 (SimInstance.member): device
memory per member next to the shared synapse tables, and one assimilation
window (100 ms of biological time per member, conductances of two targets
resampled per member as assim.cpp:94-103 does) for M members in turn.

    python tools/ensemble_capacity.py [--members M] [--window-steps S]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import torch  # noqa: E402

from paper_2308_01241_b200 import netgen  # noqa: E402
from paper_2308_01241_b200.engine import SimOptions  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--members", type=int, default=8)
    ap.add_argument("--window-steps", type=int, default=100)
    a = ap.parse_args()
    net = netgen.build_network(bench.workload_cfg())
    opt = SimOptions(steps=a.window_steps, record_raster=False, record_timings=False)
    torch.cuda.synchronize()
    f0 = torch.cuda.mem_get_info()[0]
    donor = netgen.GeneratedSimInstance(net, opt)
    f1 = torch.cuda.mem_get_info()[0]
    members = [donor.member() for _ in range(a.members)]
    f2 = torch.cuda.mem_get_info()[0]
    units = net.arrays["units"]
    conds = []  # per member: AMPA scales of two excitatory units (vectorised sampler)
    for m in range(a.members):
        salt = netgen.mix_key(m + 1, 1)
        conds.append([(u, netgen.sample_conductances(5, salt, u, 0, -1.65, 0.2,
                                                      int(units[u]["neurons"])))
                      for u in (0, 2)])
    for m, sim in enumerate(members):  # warm-up window
        for u, v in conds[m]:
            sim.set_conductances(u, 0, v)
        sim.advance(a.window_steps)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev_ms, events = 0.0, 0
    for m, sim in enumerate(members):
        for u, v in conds[m]:
            sim.set_conductances(u, 0, v)
        r = sim.advance(a.window_steps)
        dev_ms += r.device_ms
        events += r.events
    wall = time.perf_counter() - t0
    print(json.dumps({
        "workload": "config2 ensemble (1M neurons, K=1000, 1e9 synapses per member)",
        "members": a.members, "window_bio_ms": a.window_steps,
        "tables_and_donor_gb": (f0 - f1) / 1e9, "per_member_gb": (f1 - f2) / 1e9 / a.members,
        "members_fitting_180gb_estimate": int((180e9 - (f0 - f1)) / max(1, (f1 - f2) / a.members)),
        "window_wall_s_all_members": wall, "device_s": dev_ms / 1e3,
        "events_per_s": events / wall}), flush=True)


if __name__ == "__main__":
    main()
