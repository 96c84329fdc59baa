"""Benchmark of the B200 simulation step on BASELINE.json's config 2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1]): 1M conductance-LIF neurons (ring of 100
voxels x 10 000, subcortex, 80% E / 20% I), in-degree K = 1000 (1e9 synapses,
4 receptor types), dt = 1 ms, seed 2, ~10 Hz mean rate (g_location[AMPA] and
ou_mean calibrated with tools/calibrate_rate.py; the reference defaults are
bistable at K = 1000).  Synthetic network drawn by the
reference's own sampler, on the device.

One bench step = one SimInstance::advance of `--bio-ms` milliseconds of
biological time (default 100 ms = 100 dt-steps).  Metric: synaptic events per
second (events = delivered table entries, (gating_inner + gating_outer) / 2,
engine.cpp:459-463); wall seconds per biological second is reported beside it.

`value` uses the device time of the step kernel (CUDA events on the engine's
launching stream), inputs resident in HBM.  `e2e` times each step as the
assimilation caller drives the C ABI (assim.cpp:91-107): set_conductances of
every local unit from pinned host buffers (the host->device bytes), then a
synchronous advance whose results (rates, FLOP tallies, timing rows) are
copied back to host memory (the device->host bytes).  The
synapse tables (12 GB) exceed L2 (126 MB), so no flush is needed.

--impl reference runs the reference CPU engine (oracle/_ref/libvoxsim_ref.so,
built from /root/reference/proj/src) on a bounded, down-scaled sample of the
same workload (same K, parameters, dt and operating point; fewer voxels) with
scheduler "threads" on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

G_LOC_10HZ = [-2.3, -4.1997, -0.2231, -2.9957]
OU_MEAN_10HZ = 275.0
SEED = 2
# K = 500 operating points (tools/calibrate_rate.py, ring 100 x 10 000):
# rate -> (g_location[AMPA], ou_mean); measured 7.5 / 10.0 / 15.2 / 29.9 Hz
K500_POINTS = {7: (-2.0, 250.0), 10: (-2.2, 275.0), 15: (-1.9, 275.0), 30: (-2.0, 325.0)}


def workload_cfg(voxels=100, npv=10000, k_in=1000, dt_ms=1.0, workers=1):
    return {"seed": SEED, "dt_ms": dt_ms, "steps": 1000, "workers": workers,
            "connectome": {"kind": "ring", "voxels": voxels, "neurons_per_voxel": npv},
            "partition": {"method": "sequential" if workers == 1 else "greedy"},
            "regions": {"subcortex": {"k_in": k_in, "g_location": G_LOC_10HZ,
                                      "ou_mean": OU_MEAN_10HZ}}}


def dti_cfg(workers=1, rate=10, dt_ms=1.0, total=20_000_000):
    """Config 3 / 4: 200-voxel DTI-like network, lognormal voxel sizes,
    20M neurons, K = 500 (1e10 synapses), greedy partition under the B200
    byte model (strong scaling over GPUs)."""
    from paper_2308_01241_b200 import netgen
    path = ROOT / "build" / f"dti200_{total}.txt"
    if not path.exists():  # every rank may get here: write privately, rename atomically
        path.parent.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(f".{os.getpid()}.tmp")
        netgen.write_connectome_file(netgen.dti_like_connectome(total_neurons=total), tmp)
        os.replace(tmp, path)
    ampa, ou = K500_POINTS[rate]
    return {"seed": SEED, "dt_ms": dt_ms, "steps": 1000, "workers": workers,
            "connectome": {"kind": "file", "path": str(path)},
            "partition": {"method": "greedy", "byte_model": "b200"},
            "regions": {"subcortex": {"k_in": 500, "g_location": [ampa] + G_LOC_10HZ[1:],
                                      "ou_mean": ou}}}


def config5_cfg(workers=1, dt_ms=1.0, per_gpu=25_000_000, rate=15):
    """Config 5: the whole-box network, 1000-voxel DTI-like connectome with
    lognormal voxel sizes, K = 500, ~15 Hz, 25M neurons per GPU (2e8 neurons
    and 1e11 synapses on 8 GPUs, 150 GB of synapse table per GPU), greedy
    partition under the B200 byte model.  Weak-scaled: --gpus N simulates
    N x 25M neurons."""
    from paper_2308_01241_b200 import netgen
    total = per_gpu * workers
    path = ROOT / "build" / f"dti1000_{total}.txt"
    if not path.exists():
        path.parent.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(f".{os.getpid()}.tmp")
        netgen.write_connectome_file(
            netgen.dti_like_connectome(voxels=1000, total_neurons=total), tmp)
        os.replace(tmp, path)
    ampa, ou = K500_POINTS[rate]
    return {"seed": SEED, "dt_ms": dt_ms, "steps": 1000, "workers": workers,
            "connectome": {"kind": "file", "path": str(path)},
            "partition": {"method": "greedy", "byte_model": "b200"},
            "regions": {"subcortex": {"k_in": 500, "g_location": [ampa] + G_LOC_10HZ[1:],
                                      "ou_mean": ou}}}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def ensure_world(args) -> None:
    """`--gpus N` means N ranks, one per GPU.  Launched by torchrun the world
    size must match; launched bare with N > 1, re-launch this command under
    torch.distributed.run (127.0.0.1 rendezvous) and exit with its status."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
        return
    if args.gpus <= 1:
        return
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    raise SystemExit(subprocess.call(cmd))


def host_cores() -> dict:
    """Host CPU inventory for the CPU-baseline records: logical CPUs usable by
    this process, and physical cores (distinct (package, core) pairs)."""
    try:
        logical = len(os.sched_getaffinity(0))
    except AttributeError:
        logical = os.cpu_count() or 1
    phys = set()
    try:
        pkg = core = None
        for line in open("/proc/cpuinfo"):
            if line.startswith("physical id"):
                pkg = line.split(":")[1].strip()
            elif line.startswith("core id"):
                core = line.split(":")[1].strip()
            elif not line.strip():
                if core is not None:
                    phys.add((pkg, core))
                pkg = core = None
        if core is not None:
            phys.add((pkg, core))
    except OSError:
        pass
    return {"nproc": logical, "physical_cores": len(phys) or None}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every ~5 ms during
    the timed region through NVML (the counters nvidia-smi reads); falls
    back to `nvidia-smi -lms 100` when NVML is unavailable."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    BITS = (0x8, 0x40, 0x20, 0x4)  # nvmlClocksEventReason* masks

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.sm, self.mx, self.reasons = [], [], set()
        self.proc = None
        self.stop = threading.Event()
        self.t = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            p = torch.cuda.get_device_properties(self.gpu)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def _poll(self, nv, h):
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            self.mx.append(float(mx))
            r = get_r(h)
            self.reasons.update(n for n, b in zip(self.NAMES, self.BITS) if r & b)
            self.stop.wait(0.005)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self.t = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.t.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            if r[1].replace(".", "").isdigit():
                self.sm.append(float(r[1]))
            if r[2].replace(".", "").isdigit():
                self.mx.append(float(r[2]))
            self.reasons.update(n for i, n in enumerate(self.NAMES)
                                if len(r) > 5 + i and r[5 + i].lower() == "active")

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=5)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx or [0.0]),
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(workload: str, ws: int, kernel: str):
    """DRAM bytes per launch of `kernel` from a committed `ncu --set full`
    capture of this same workload and GPU count (profiles/traffic.json:
    {"<workload>/n<ws>/<kernel>": {"dram_bytes_per_launch": ...}}), else None."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        rec = json.loads(p.read_text()).get(f"{workload}/n{ws}/{kernel}")
        return rec.get("dram_bytes_per_launch") if rec else None
    except Exception:
        return None


class CpuReference:
    """The reference engine on a down-scaled sample of the workload: same K,
    parameters, dt and operating point, fewer voxels."""

    def __init__(self, sample_voxels: int, threads: int):
        sys.path.insert(0, str(ROOT / "tests"))
        from refnet import RefNet, RefSim
        from paper_2308_01241_b200.engine import SimOptions
        self.workers = max(1, min(threads, 2 * sample_voxels))
        cfg = workload_cfg(voxels=sample_voxels, workers=self.workers)
        cfg["scheduler"] = "threads"
        self.net = RefNet(cfg)
        self.sim = RefSim(self.net, SimOptions(dt_ms=cfg["dt_ms"], record_raster=False,
                                               record_timings=False),
                          scheduler="threads" if self.workers > 1 else "loopback")
        self.neurons = self.net.total_neurons
        self.threads = 3 * self.workers if self.workers > 1 else 1

    def step(self, steps: int):
        r = self.sim.advance(steps)
        events = (r.flops["gating_inner"] + r.flops["gating_outer"]) // 2
        return events, r.seconds, r.total_spikes


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    hc = host_cores()
    ref = CpuReference(args.cpu_voxels, args.cpu_workers or hc["nproc"])
    # size each bench step so the whole warmup + steps run takes about
    # --cpu-budget-s on this host (host core counts differ between boxes)
    e0, s0, _ = ref.step(200)
    per_step_s = args.cpu_budget_s / max(1, args.steps + args.warmup)
    args.cpu_steps = int(min(args.cpu_steps, max(50, per_step_s / max(s0 / 200, 1e-9))))
    for _ in range(args.warmup):
        ref.step(args.cpu_steps)
    ev = sec = spk = 0
    for _ in range(args.steps):
        e, s, k = ref.step(args.cpu_steps)
        ev, sec, spk = ev + e, sec + s, spk + k
    value = ev / sec
    rate = spk / (ref.neurons * args.steps * args.cpu_steps * 1e-3)
    sample = (f"ring {args.cpu_voxels} voxels x 10000 neurons, K=1000, dt=1 ms, "
              f"{args.cpu_steps} steps per bench step, {ref.workers} workers "
              f"(scheduler threads: {ref.threads} engine threads on {hc['nproc']} CPUs), "
              f"{rate:.1f} Hz")
    line = {"metric": "synaptic_events_per_s", "value": value, "unit": "events/s",
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sec / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 state / i64 Q16 / f64 noise",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "config2-sample", "neurons": ref.neurons, "k_in": 1000,
                       "dt_ms": 1.0, "parallelism": f"cpu threads x{ref.threads}"},
            "wall_s_per_bio_s_extrapolated_1M": (sec / args.steps) / (args.cpu_steps * 1e-3)
            * (1e6 / ref.neurons),
            "cpu_baseline": {"value": value, "unit": "events/s", "cores": hc["nproc"],
                             "nproc": hc["nproc"], "physical_cores": hc["physical_cores"],
                             "engine_workers": ref.workers, "engine_threads": ref.threads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import numpy as np
    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("gloo")
        dist = tdist
    from paper_2308_01241_b200 import netgen
    from paper_2308_01241_b200.engine import SimOptions

    dev = local if ws > 1 else args.device
    bio_steps = int(round(args.bio_ms / args.dt))
    if args.workload == "config2":
        # weak scaling: 100 voxels x 10 000 neurons per GPU, one worker per rank,
        # contiguous voxel blocks (sequential partition of the ring)
        cfg = workload_cfg(voxels=100 * ws, dt_ms=args.dt, workers=ws)
        if ws > 1:
            cfg["partition"]["method"] = "sequential"
    elif args.workload == "config5":  # weak scaling: 25M neurons per GPU, K = 500, 15 Hz
        cfg = config5_cfg(workers=ws, dt_ms=args.dt, per_gpu=args.neurons or 25_000_000,
                          rate=args.rate if args.rate != 10 else 15)
    else:  # config3 (10 Hz) / config4 rate sweep: strong scaling, 20M neurons
        cfg = dti_cfg(workers=ws, rate=args.rate, dt_ms=args.dt,
                      total=args.neurons or 20_000_000)
    if args.workload != "config2":
        cfg["partition"]["byte_model"] = args.byte_model
    net = netgen.build_network(cfg)
    # the reference arm's options (record_raster / record_timings off): the
    # per-step wire-byte rows would add a spike-log readback per advance
    opt = SimOptions(steps=bio_steps, dt_ms=args.dt, record_raster=False, record_timings=False,
                     device=dev)
    if ws > 1:
        sim = netgen.DistributedSimInstance(net, opt, rank, ws)
    else:
        sim = netgen.GeneratedSimInstance(net, opt)
    import torch
    free_b, total_b = torch.cuda.mem_get_info(dev)
    mem_used = float(total_b - free_b)
    # e2e input per step, as the assimilation caller feeds the boundary
    # (assim.cpp:91-107, EnsembleMember::run_window): fresh AMPA conductance
    # scales for every local unit from pinned host buffers, staged by
    # set_conductances and uploaded by the following advance.  Two windows'
    # worth are drawn up front (sample_conductances with the assimilation
    # salt, netgen.cpp:318-329) and alternated; g_location/g_scale are the
    # population's own, so the operating point is unchanged.
    import torch
    windows = []
    for w in range(2):
        sets = []
        salt = netgen.mix_key(1, w + 1)
        for u, unit in enumerate(net.layout.units):
            if unit.neurons == 0 or (ws > 1 and net.unit_worker[u] != rank):
                continue
            pop = net.layout.pop_of_unit(u)
            buf = torch.empty(unit.neurons, dtype=torch.float32, pin_memory=True).numpy()
            buf[:] = netgen.sample_conductances(SEED, salt, u, 0, pop.g_location[0],
                                                pop.g_scale[0], unit.neurons)
            sets.append((u, buf))
        windows.append(sets)

    # one boundary crossing per window: set_conductances of every local unit
    # (vxb_set_conductances_batch, item-by-item semantics, copies on the
    # host cores)
    from paper_2308_01241_b200.engine import ConductanceBatch
    batches = [ConductanceBatch([(u, 0, buf) for u, buf in w]) for w in windows]

    def feed(i):
        sim.set_conductances_batch(batches[i % 2])

    for i in range(args.warmup):
        feed(i)
        sim.advance(bio_steps)

    def barrier():
        if dist:
            dist.barrier()

    dev_ms, wall, events, spikes, h2d, d2h, launches, results = [], [], 0, 0, 0, 0, 0, []
    xwait, xarr, stage_s = 0.0, 0.0, 0.0
    with ClockSampler(dev) as clk:
        barrier()
        t_all = time.perf_counter()
        for _ in range(args.steps):
            t0 = time.perf_counter()
            feed(_)
            stage_s += time.perf_counter() - t0
            r = sim.advance(bio_steps)  # synchronous C-ABI call, results on host
            wall.append(time.perf_counter() - t0)
            dev_ms.append(r.device_ms)
            events += r.events
            spikes += r.total_spikes
            h2d += r.h2d_bytes
            d2h += r.d2h_bytes
            launches += r.launches
            xwait += r.exchange_wait_ms
            xarr += r.exchange_arrival_ms
        barrier()
        t_all = time.perf_counter() - t_all
    schedule = sim.schedule_info()
    sim.close()
    dev_s = sum(dev_ms) / 1e3
    wall_s = sum(wall)
    # max over ranks of time, sum of work
    if dist:
        import torch
        t = torch.tensor([dev_s, wall_s, xwait, xarr, stage_s, mem_used], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, wall_s, xwait, xarr, stage_s, mem_used = (float(x) for x in t)
        e = torch.tensor([events, spikes, launches], dtype=torch.float64)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        events, spikes, launches = (int(x) for x in e)
    if rank != 0:
        return
    n = net.total_neurons
    bio_s = args.steps * bio_steps * args.dt * 1e-3
    value = events / dev_s
    rate = spikes / (n * bio_s)
    # roofline of the step kernel: algorithmic bytes, per GPU
    neuron_steps = n * args.steps * bio_steps
    alg_bytes = (98 * neuron_steps + 12 * events + 20 * spikes) / ws
    peak, peak_kind = measured_peak_hbm()
    achieved = alg_bytes / dev_s / 1e9
    # per advance and rank: one conductance-scatter launch (the staged
    # set_conductances), one scratch-clearing launch + the step kernel launch(es)
    launches_per = max(1, launches // max(1, args.steps * ws) - 2)
    if args.workload == "config2":
        wl = "config2" if ws == 1 else f"config2 x{ws} (ring {100 * ws} voxels)"
    elif args.workload == "config5":
        wl = (f"config5 ({net.total_neurons} neurons, 1000-voxel DTI-like, K=500, "
              f"{args.rate if args.rate != 10 else 15} Hz point)")
    else:
        wl = (f"{args.workload} (200-voxel DTI-like, {net.total_neurons} neurons, "
              f"K=500, {args.rate} Hz point)")
    kernel = schedule.get("kernel", "vxb::step_kernel")
    traffic = ncu_traffic(args.workload, ws, kernel)
    line = {
        "metric": "synaptic_events_per_s", "value": value, "unit": "events/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.workload in ("config2", "config5") else "strong",
        "vs_baseline": None,
        "dtype": "f32 state / i64 Q16 / f64 noise", "data": "synthetic",
        "config": {"workload": wl,
                   "neurons_per_gpu": net.total_neurons // ws,
                   "synapses_per_gpu": net.synapse_count // ws,
                   "k_in": 1000 if args.workload == "config2" else 500, "dt_ms": args.dt,
                   "bio_ms_per_step": args.bio_ms, "seed": SEED,
                   "parallelism": f"neuron shards x{ws}, NVLink spike exchange" if ws > 1
                   else "single",
                   "l2": f"inputs larger than L2 ({12 * net.synapse_count / ws / 1e9:.0f} GB "
                         "synapse table per GPU)",
                   "schedule": schedule},
        "wall_s_per_bio_s": dev_s / bio_s,
        # exchange (max over ranks, per simulated step): the time CTAs spun
        # on a peer's flag once their local work was done, and how long after
        # the phase start the last peer's batch arrived
        "exposed_exchange_us_per_step": 1e3 * xwait / (args.steps * bio_steps) if ws > 1 else 0.0,
        "exchange_arrival_lag_us_per_step": 1e3 * xarr / (args.steps * bio_steps) if ws > 1 else 0.0,
        "mean_rate_hz": rate,
        "device_memory_used_gb": mem_used / 1e9,  # max over ranks, after load
        "events_per_s_per_gpu": value / ws,
        "e2e": {"value": events / wall_s, "unit": "events/s",
                "h2d_bytes_per_step": h2d // max(1, args.steps * ws),
                "d2h_bytes_per_step": d2h // max(1, args.steps * ws),
                "wall_s_per_bio_s": wall_s / bio_s,
                "host_stage_ms_per_step": 1e3 * stage_s / args.steps},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": kernel,
                     "alg_bytes_per_launch": alg_bytes / max(1, launches_per * args.steps),
                     "exchange": "4 B per (spike, destination GPU) over NVLink" if ws > 1 else None,
                     "model": "98 B/neuron-step + 12 B/event + 20 B/delivered spike"},
        # the resource that bounds delivery: scattered L2 red.add, measured
        # ceiling 1.93e11/s per GPU (profiles/r01_delivery_ceiling.txt)
        "roofline_atomic": {"bound": "l2_atomic", "achieved": value / ws, "peak": 1.93e11,
                            "unit": "red.add/s per GPU", "frac": value / ws / 1.93e11,
                            "peak_kind": "measured (tools/microbench_delivery.cu)"},
        "clocks": clk.summary(),
    }
    if not args.no_cpu and args.workload == "config2":
        try:
            ref = CpuReference(args.cpu_voxels, args.cpu_workers or host_cores()["nproc"])
            _, s0, _ = ref.step(300)  # warm-up + rate probe: ~cpu_sample_seconds of sample
            n_s = int(min(args.cpu_sample_steps,
                          max(500, args.cpu_sample_seconds / max(s0 / 300, 1e-9))))
            args.cpu_sample_steps = n_s
            e, s, k = ref.step(n_s)
            hc = host_cores()
            line["cpu_baseline"] = {
                "value": e / s, "unit": "events/s", "cores": hc["nproc"],
                "nproc": hc["nproc"], "physical_cores": hc["physical_cores"],
                "engine_workers": ref.workers, "engine_threads": ref.threads,
                "kind": "reference",
                "sample": f"ring {args.cpu_voxels}x10000 neurons, K=1000, {args.cpu_sample_steps} "
                          f"steps, {ref.workers} workers (scheduler threads: {ref.threads} "
                          f"engine threads on {hc['nproc']} CPUs), "
                          f"{k / (ref.neurons * args.cpu_sample_steps * 1e-3):.1f} Hz, "
                          f"{s:.1f} s wall"}
        except Exception as e:  # the checker is optional on the GPU arm
            line["cpu_baseline"] = {"value": None, "unit": "events/s", "cores": 0,
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--bio-ms", type=float, default=100.0)
    ap.add_argument("--dt", type=float, default=1.0)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--cpu-voxels", type=int, default=12)
    ap.add_argument("--cpu-steps", type=int, default=4000,
                    help="--impl reference: simulated steps per bench step")
    ap.add_argument("--cpu-sample-steps", type=int, default=12000,
                    help="cpu_baseline of the B200 arm: at most this many simulated steps")
    ap.add_argument("--cpu-sample-seconds", type=float, default=15.0,
                    help="cpu_baseline of the B200 arm: target wall time of the sample")
    ap.add_argument("--cpu-budget-s", type=float, default=150.0,
                    help="--impl reference: target wall time of warmup + steps")
    ap.add_argument("--cpu-workers", type=int, default=0,
                    help="reference engine workers (0: one per host core, at most 2 per sample voxel)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="config2",
                    choices=["config2", "config3", "config4", "config5"])
    ap.add_argument("--rate", type=int, default=10, choices=[7, 10, 15, 30],
                    help="config3/4 operating point (Hz)")
    ap.add_argument("--neurons", type=int, default=0,
                    help="config3/4 network size (default 20M); config5 neurons per GPU (25M)")
    ap.add_argument("--byte-model", default="b200", choices=["b200", "b200_time"],
                    help="config3/4/5 partition: HBM bytes (default) or the B200 time model")
    args = ap.parse_args()
    ensure_world(args)
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
