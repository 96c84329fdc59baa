"""Generate the golden fixtures in tests/golden/ from the reference build.

    python tests/golden/make_golden.py

Every value is produced by the UNMODIFIED reference engine
(oracle/_ref/libvoxsim_ref.so, built from /root/reference/proj/src by
oracle/Makefile) through its own API, so the fixtures pin the oracle and the
CUDA engine without /root/reference being present (e.g. on the GPU box).
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))

from paper_2308_01241_b200.engine import ForcedSpike, SimOptions  # noqa: E402
from refnet import RefNet, RefSim, make_config, ref_lib  # noqa: E402

L = ref_lib()

# --- rng (test_rng.cpp:13-35 plus a wider sweep) ---------------------------
rng = {
    "stream_word": [[b, k, L.ref_stream_word(b, k)] for b, k in
                    [(0, 0), (0, 1), (1, 0), (0xdeadbeef, 7), (123456789, 1000000)]],
    "stream_u01": [[42, k, L.ref_stream_u01(42, k).hex()] for k in range(4)],
    "mix_key": [[a, b, L.ref_mix_key2(a, b)] for a in (0, 1, 5, 2**63 + 3) for b in (0, 1, 17, 2**40)],
    "stream_below": [[L.ref_mix_key2(11, 4), k, 7, L.ref_stream_below(L.ref_mix_key2(11, 4), k, 7)]
                     for k in range(16)],
    "stream_normal": [[L.ref_mix_key3(5, 1, 17), k, L.ref_stream_normal(L.ref_mix_key3(5, 1, 17), k).hex()]
                      for k in range(64)],
    "quantize": [[w, L.ref_quantize_weight(w)] for w in (0.0, -3.5, 1.0, 0.013, 0.55, 1.2345, 7.77, 0.9999847, 1.00000762939453125)],
}
(HERE / "rng.json").write_text(json.dumps(rng, indent=1))

# --- OU noise samples as the engine consumes them (engine.cpp:551-553) -----
seeds = np.array([1, 2, 1401], np.uint64)
gids = np.arange(0, 4096, 7, dtype=np.uint64)
steps = np.arange(0, 2048, 13, dtype=np.uint64)
xi = np.zeros((len(seeds), len(gids), len(steps)), np.float32)
for a, s in enumerate(seeds):
    for b, g in enumerate(gids):
        for c, t in enumerate(steps):
            xi[a, b, c] = L.ref_ou_xi(int(s), int(g), int(t))
np.savez_compressed(HERE / "xi.npz", seeds=seeds, gids=gids, steps=steps, xi=xi)

# --- small engine runs -------------------------------------------------------
def run(name, cfg, opt, even=0, steps=None):
    net = RefNet(cfg, even_workers=even)
    r = RefSim(net, opt).advance(steps or opt.steps)
    keys = np.array(sorted(zip(r.raster["step"].tolist(), r.raster["gid"].tolist())), np.uint64).reshape(-1, 2)
    np.savez_compressed(HERE / f"{name}.npz", raster=keys, rates=r.rates, probe_v=r.probe_v,
                        probe_i=r.probe_i, flops=np.array(list(r.flops.values()), np.uint64),
                        total=np.uint64(r.total_spikes), cfg=json.dumps(cfg), even=even,
                        probe_gids=np.array(list(opt.probe_gids), np.uint64))
    return r.total_spikes

counts = {}
counts["six_neurons"] = run("six_neurons", make_config(seed=91, voxels=1, npv=6, k_in=2),
                            SimOptions(steps=150, probe_gids=list(range(6))))
counts["ring3_w3"] = run("ring3_w3", make_config(seed=5, voxels=3, npv=60, k_in=8, rho=0.4),
                         SimOptions(steps=120, probe_gids=[7, 179]), even=3)
counts["hot_forced"] = run("hot_forced", make_config(seed=3, voxels=1, npv=8, k_in=2, ou_mean=400.0, ou_sigma=150.0),
                           SimOptions(steps=30, forced_spikes=[ForcedSpike(4, 2)], probe_gids=[2]))
# survey goldens: spike totals only
net = RefNet(make_config(seed=1, voxels=1, npv=10000, k_in=100, dt_ms=0.1, steps=10000))
counts["config1_dt0.1_10000"] = RefSim(net, SimOptions(steps=10000, dt_ms=0.1, record_raster=False)).advance(10000).total_spikes
net = RefNet(make_config(seed=1, voxels=1, npv=10000, k_in=100, dt_ms=1.0, steps=1000))
counts["config1_dt1_1000"] = RefSim(net, SimOptions(steps=1000, dt_ms=1.0, record_raster=False)).advance(1000).total_spikes
(HERE / "counts.json").write_text(json.dumps(counts, indent=1))
print(counts)
