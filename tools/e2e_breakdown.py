"""Where the end-to-end time of one bench step goes (config 2, 1 GPU): host
staging of the conductances, the C-ABI advance (H2D + kernel + readback), and
the Python-side result marshalling, against the device-timed kernel."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2308_01241_b200 import netgen  # noqa: E402
from paper_2308_01241_b200.engine import ConductanceBatch, SimOptions  # noqa: E402

cfg = bench.workload_cfg()
net = netgen.build_network(cfg)
opt = SimOptions(steps=100, record_raster=False, record_timings=False)
sim = netgen.GeneratedSimInstance(net, opt)
import torch  # noqa: E402
sets = []
for u, unit in enumerate(net.layout.units):
    pop = net.layout.pop_of_unit(u)
    buf = torch.empty(unit.neurons, dtype=torch.float32, pin_memory=True).numpy()
    buf[:] = netgen.sample_conductances(bench.SEED, netgen.mix_key(1, 1), u, 0, pop.g_location[0],
                                        pop.g_scale[0], unit.neurons)
    sets.append((u, 0, buf))
batch = ConductanceBatch(sets)
inner = getattr(sim, "_sim", sim)
rows = []
for k in range(23):
    t0 = time.perf_counter()
    sim.set_conductances_batch(batch)
    t1 = time.perf_counter()
    inner.advance(100, fetch=False)
    t2 = time.perf_counter()
    r = inner.result()
    t3 = time.perf_counter()
    if k >= 3:
        rows.append((t1 - t0, t2 - t1, t3 - t2, r.device_ms * 1e-3))
a = np.array(rows) * 1e3
print("per 100-step advance (ms): stage %.3f | vxb_advance %.3f | result() %.3f | device kernel %.3f"
      % tuple(a.mean(0)))
print("advance overhead beyond the kernel: %.3f ms" % (a[:, 1] - a[:, 3]).mean())
