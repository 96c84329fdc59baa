"""Cost of the e2e host stage: set_conductances of every config-2 unit
(200 x 10 000 floats from pinned buffers) per step, split into the Python
binding and the C ABI call."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_01241_b200 import netgen  # noqa: E402
from paper_2308_01241_b200.engine import SimOptions  # noqa: E402

net = netgen.build_network(bench.workload_cfg())
sim = netgen.GeneratedSimInstance(net, SimOptions(steps=10, record_raster=False))
units = [(u, int(x["neurons"])) for u, x in enumerate(net.arrays["units"]) if x["neurons"]]
bufs = [(u, torch.empty(n, dtype=torch.float32, pin_memory=True).numpy()) for u, n in units]
for _, b in bufs:
    b[:] = 1.0
for rep in range(3):
    t0 = time.perf_counter()
    for u, b in bufs:
        sim.set_conductances(u, 0, b)
    t1 = time.perf_counter()
    addrs = [(u, C.addressof(C.c_char.from_buffer(b)), b.size) for u, b in bufs]
    f = sim._lib.vxb_set_conductances
    t2 = time.perf_counter()
    for u, a, n in addrs:
        f(sim._h, u, 0, a, n)
    t3 = time.perf_counter()
    sim.advance(1)
    print(f"python API {1e3 * (t1 - t0):.3f} ms, raw C ABI {1e3 * (t3 - t2):.3f} ms "
          f"for {len(bufs)} units, {sum(n for _, n in units) * 4 / 1e6:.1f} MB")
