"""Python mirror of the reference host API for the simulation step.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/voxsim/engine.hpp (SimOptions, RunResult,
SimInstance, run_simulation) and util.hpp (ConfigError, SimError), so the
parity tests read like the reference's own tests (test_engine.cpp).  Every
call goes through the C ABI in include/vxb.h (libvxb.so); nothing here
computes simulation results.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _abi
from ._abi import (FORCED_DTYPE, INJECTION_DTYPE, NEURON_DTYPE, RASTER_DTYPE, SYN_DTYPE,
                   TIMINGS_DTYPE, UNIT_DTYPE, ptr)


class ConfigError(RuntimeError):
    """voxsim::ConfigError (util.hpp:14-16)."""


class SimError(RuntimeError):
    """voxsim::SimError (util.hpp:19-21)."""


def _raise(rc: int, msg: str):
    if rc == _abi.VXB_ECONFIG:
        raise ConfigError(msg)
    if rc == _abi.VXB_ESIM:
        raise SimError(msg)
    raise RuntimeError(f"vxb error {rc}: {msg}")


# ------------------------------------------------------------------ tables
@dataclass
class WorkerTable:
    """voxsim::WorkerTable (netgen.hpp:55-64) as numpy arrays in vxb.h layout."""
    worker: int
    worker_count: int
    seed: int
    neurons: np.ndarray      # NEURON_DTYPE [n]
    synapses: np.ndarray     # SYN_DTYPE [nsyn], rows by target
    row_base: np.ndarray     # uint64 [n+1]


@dataclass
class NetworkTables:
    """voxsim::NetworkTables + the NetworkLayout units the engine needs."""
    workers: List[WorkerTable]
    unit_worker: np.ndarray      # uint16 [units]
    unit_local_base: np.ndarray  # uint32 [units]
    units: np.ndarray            # UNIT_DTYPE [units]
    n_voxels: int

    @property
    def total_neurons(self) -> int:
        return int(sum(w.neurons.shape[0] for w in self.workers))

    @property
    def synapse_count(self) -> int:
        return int(sum(w.synapses.shape[0] for w in self.workers))

    def _descriptor(self):
        wt = (_abi.WorkerTable * len(self.workers))()
        for i, w in enumerate(self.workers):
            assert w.neurons.dtype == NEURON_DTYPE and w.synapses.dtype == SYN_DTYPE
            wt[i] = _abi.WorkerTable(w.worker, w.worker_count, w.neurons.shape[0], w.seed,
                                     w.synapses.shape[0], ptr(w.neurons), ptr(w.synapses),
                                     ptr(w.row_base))
        net = _abi.Network(len(self.workers), self.units.shape[0], self.n_voxels, 0,
                           C.cast(wt, C.POINTER(_abi.WorkerTable)), ptr(self.unit_worker),
                           ptr(self.unit_local_base), ptr(self.units))
        return net, wt


# ----------------------------------------------------------------- options
@dataclass
class Injection:
    """voxsim::Injection (engine.hpp:16-21)."""
    from_step: int = 0
    to_step: int = 0
    voxel: int = 0
    current_pa: float = 0.0


@dataclass
class ForcedSpike:
    """voxsim::ForcedSpike (engine.hpp:25-28)."""
    step: int = 0
    gid: int = 0


@dataclass
class SimOptions:
    """voxsim::SimOptions (engine.hpp:30-45).  scheduler "cuda" is the B200
    engine; "threads"/"loopback" are accepted and run the same engine."""
    steps: int = 0
    dt_ms: float = 1.0
    scheduler: str = "cuda"
    transport: str = "queue"
    workers_per_node: int = 4
    recv_timeout_ms: int = 30000
    record_raster: bool = True
    record_timings: bool = True
    probe_gids: Sequence[int] = field(default_factory=list)
    injections: Sequence[Injection] = field(default_factory=list)
    forced_spikes: Sequence[ForcedSpike] = field(default_factory=list)
    device: int = -1
    n_devices: int = 1

    def _descriptor(self):
        probes = np.asarray(list(self.probe_gids), dtype=np.uint64)
        inj = np.zeros(len(self.injections), INJECTION_DTYPE)
        for i, x in enumerate(self.injections):
            inj[i] = (x.from_step, x.to_step, x.voxel, x.current_pa)
        forced = np.zeros(len(self.forced_spikes), FORCED_DTYPE)
        for i, x in enumerate(self.forced_spikes):
            forced[i] = (x.step, 0, x.gid)
        keep = (probes, inj, forced, self.scheduler.encode(), self.transport.encode())
        o = _abi.Options(self.dt_ms, keep[3], keep[4], self.workers_per_node, 0,
                         self.recv_timeout_ms, int(self.record_raster),
                         int(self.record_timings), ptr(probes), probes.size, inj.size,
                         ptr(inj), ptr(forced), forced.size, self.device, self.n_devices, 0)
        return o, keep


# ------------------------------------------------------------------ result
@dataclass
class ProbeTrace:
    """voxsim::ProbeTrace (engine.hpp:47-53)."""
    gid: int
    v: np.ndarray
    i_syn: np.ndarray


@dataclass
class RateSeries:
    """voxsim::RateSeries (stats.hpp:93-105) with the same rate helpers."""
    steps: int
    dt_ms: float
    unit_neurons: np.ndarray
    counts: np.ndarray  # [units][steps] uint32

    def rate_hz(self, unit: int, step: int) -> float:
        n = int(self.unit_neurons[unit])
        return 0.0 if n == 0 else self.counts[unit, step] / (n * self.dt_ms * 1e-3)

    def network_mean_hz(self, from_step: int = 0) -> float:
        if from_step >= self.steps:
            return 0.0
        total_n = int(self.unit_neurons.sum())
        if total_n == 0:
            return 0.0
        spikes = int(self.counts[:, from_step:].sum())
        return spikes / (total_n * (self.steps - from_step) * self.dt_ms * 1e-3)

    def voxel_counts(self, unit_voxel: np.ndarray, n_voxels: int, step: int) -> np.ndarray:
        out = np.zeros(n_voxels, np.uint32)
        np.add.at(out, unit_voxel, self.counts[:, step])
        return out


@dataclass
class HemoParams:
    """voxsim::HemoParams (hemo.hpp:10-23): Balloon-Windkessel constants."""
    kappa: float = 0.65   # signal decay, 1/s
    gamma: float = 0.41   # flow-dependent elimination, 1/s
    tau: float = 0.98     # hemodynamic transit time, s
    alpha: float = 0.32   # Grubb's exponent
    e0: float = 0.34      # resting oxygen extraction
    v0: float = 0.02      # resting venous volume fraction

    def k1(self) -> float:
        return 7.0 * self.e0

    def k2(self) -> float:
        return 2.0

    def k3(self) -> float:
        return 2.0 * self.e0 - 0.2

    def _c(self) -> _abi.HemoParams:
        return _abi.HemoParams(self.kappa, self.gamma, self.tau, self.alpha, self.e0, self.v0)


HEMO_STATE_DTYPE = np.dtype([("s", "f8"), ("f", "f8"), ("v", "f8"), ("q", "f8")])


def hemo_rest(n: int) -> np.ndarray:
    """n HemoState records at rest (hemo.hpp:25-30): s = 0, f = v = q = 1."""
    st = np.zeros(n, HEMO_STATE_DTYPE)
    st["f"] = st["v"] = st["q"] = 1.0
    return st


def bold_from_drive(z, dt_s: float, sample_every: int, params: HemoParams | None = None,
                    state: np.ndarray | None = None, device: int = 0) -> np.ndarray:
    """voxsim::bold_from_drive (hemo.cpp:49-62) evaluated on the GPU for one
    drive series (1-D z) or several (2-D z[series][steps]); `state` (HEMO_STATE_DTYPE,
    one per series) is updated in place when given."""
    p = params or HemoParams()
    zz = np.ascontiguousarray(np.atleast_2d(np.asarray(z, np.float64)))
    ns, steps = zz.shape
    st = hemo_rest(ns) if state is None else state
    if st.dtype != HEMO_STATE_DTYPE or not st.flags.c_contiguous or st.size != ns:
        raise ConfigError("hemodynamics: state must be a contiguous HemoState array per series")
    out = np.zeros((ns, steps // max(1, sample_every)), np.float64)
    lib = _abi.load_library()
    rc = lib.vxb_debug_bold_from_drive(device, C.byref(p._c()), ptr(zz), steps, ns, dt_s,
                                       sample_every, ptr(st), ptr(out))
    if rc != 0:
        _raise(rc, lib.vxb_last_error(None).decode())
    return out[0] if np.ndim(z) == 1 else out


@dataclass
class RunResult:
    """voxsim::RunResult (engine.hpp:55-63)."""
    raster: np.ndarray          # RASTER_DTYPE, sorted (step, worker, local)
    timings: np.ndarray         # TIMINGS_DTYPE, sorted (step, worker)
    probes: List[ProbeTrace]
    rates: RateSeries
    flops: dict
    total_spikes: int
    steps_done: int
    device_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    launches: int = 0
    exchange_wait_ms: float = 0.0
    # BOLD-proxy readout (set_hemodynamics): [steps // sample_every][voxels],
    # and the voxel spike counts it was driven by, [steps][voxels]
    bold: np.ndarray | None = None
    voxel_counts: np.ndarray | None = None
    exchange_arrival_ms: float = 0.0

    @property
    def events(self) -> int:
        """Delivered synaptic events = (gating_inner + gating_outer) / 2."""
        return (self.flops["gating_inner"] + self.flops["gating_outer"]) // 2


# ---------------------------------------------------------------- instance
class ConductanceBatch:
    """Argument arrays of vxb_set_conductances_batch built once: (unit,
    receptor, float32 buffer) items whose buffers the caller refills."""

    def __init__(self, items):
        items = list(items)
        self.n = len(items)
        self.units = np.array([u for u, _, _ in items], np.uint32)
        self.recs = np.array([r for _, r, _ in items], np.int32)
        self.arrays = [np.ascontiguousarray(v, dtype=np.float32) for _, _, v in items]
        self.counts = np.array([a.size for a in self.arrays], np.uint32)
        self.ptrs = (C.c_void_p * max(1, self.n))(*[a.ctypes.data for a in self.arrays])
        self.units_p, self.recs_p, self.counts_p = ptr(self.units), ptr(self.recs), ptr(self.counts)


class SimInstance:
    """voxsim::SimInstance (engine.hpp:68-89) backed by the CUDA engine."""

    def __init__(self, tables: NetworkTables, options: SimOptions):
        self._lib = _abi.load_library()
        self._opt = options
        self._units = tables.units.copy()
        self._n_voxels = tables.n_voxels
        self._hemo_every = 0
        self._tables = tables
        net, keep_net = tables._descriptor()
        opt, keep_opt = options._descriptor()
        h = C.c_void_p()
        rc = self._lib.vxb_create(C.byref(net), C.byref(opt), C.byref(h))
        del keep_net, keep_opt
        if rc != 0:
            _raise(rc, self._lib.vxb_last_error(None).decode())
        self._h = h

    def _member_args(self):
        """(network descriptor, spec, keep-alive) for vxb_create_member."""
        net, keep = self._tables._descriptor()
        return C.byref(net), None, (net, keep)

    def member(self, options: SimOptions | None = None) -> "SimInstance":
        """An ensemble member (EnsembleMember, assim.cpp:74-80): a new
        instance of the same network on the same GPU that views this
        instance's synapse tables instead of building its own; its state,
        conductances and results are its own.  It keeps this instance alive."""
        opt = options or self._opt
        net, spec, keep = self._member_args()
        o, keep_opt = opt._descriptor()
        h = C.c_void_p()
        rc = self._lib.vxb_create_member(self._h, net, spec, C.byref(o), C.byref(h))
        del keep, keep_opt
        if rc != 0:
            _raise(rc, self._lib.vxb_last_error(None).decode())
        m = object.__new__(type(self))
        m.__dict__.update({k: v for k, v in self.__dict__.items() if k not in ("_h", "_donor")})
        m._opt, m._h, m._hemo_every, m._donor = opt, h, 0, self
        return m

    def close(self):
        if getattr(self, "_h", None):
            self._lib.vxb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _err(self, rc):
        _raise(rc, self._lib.vxb_last_error(self._h).decode())

    def current_step(self) -> int:
        return int(self._lib.vxb_current_step(self._h))

    def advance(self, steps: int, fetch: bool = True) -> RunResult | None:
        rc = self._lib.vxb_advance(self._h, steps)
        if rc != 0:
            self._err(rc)
        return self.result() if fetch else None

    def result(self) -> RunResult:
        L, h = self._lib, self._h
        steps = int(L.vxb_result_steps_done(h))
        nr = int(L.vxb_result_raster_size(h))
        raster = np.zeros(nr, RASTER_DTYPE)
        if nr:
            rc = L.vxb_result_raster(h, ptr(raster), nr)
            if rc:
                self._err(rc)
        nu = int(L.vxb_units(h))
        counts = np.zeros((nu, steps), np.uint32)
        if counts.size:
            L.vxb_result_rates(h, ptr(counts), counts.size)
        npb = int(L.vxb_probes(h))
        pv = np.zeros((npb, steps), np.float32)
        pi = np.zeros((npb, steps), np.float32)
        if pv.size:
            L.vxb_result_probes(h, ptr(pv), ptr(pi), pv.size)
        probes = [ProbeTrace(int(g), pv[k], pi[k]) for k, g in enumerate(self._opt.probe_gids)]
        fl = _abi.Flops()
        L.vxb_result_flops(h, C.byref(fl))
        flops = {n: int(getattr(fl, n)) for n, _ in _abi.Flops._fields_}
        nt = int(L.vxb_result_timings_size(h))
        timings = np.zeros(nt, TIMINGS_DTYPE)
        if nt:
            L.vxb_result_timings(h, ptr(timings), nt)
        rates = RateSeries(steps, self._opt.dt_ms, self._units["neurons"].astype(np.uint64),
                           counts)
        bold = vcounts = None
        if self._hemo_every:
            bold = self._bold(steps)
            vcounts = np.zeros((steps, self._n_voxels), np.uint32)
            if vcounts.size:
                L.vxb_result_voxel_counts(h, ptr(vcounts), vcounts.size)
        return RunResult(raster, timings, probes, rates, flops,
                         int(L.vxb_result_total_spikes(h)), steps,
                         float(L.vxb_result_device_ms(h)), int(L.vxb_result_h2d_bytes(h)),
                         int(L.vxb_result_d2h_bytes(h)), int(L.vxb_result_launches(h)),
                         float(L.vxb_result_exchange_wait_ms(h)), bold, vcounts,
                         float(L.vxb_result_exchange_arrival_ms(h)))

    def _bold(self, steps: int) -> np.ndarray:
        n = int(self._lib.vxb_result_bold_size(self._h))
        bold = np.zeros(n, np.float64)
        if n:
            self._lib.vxb_result_bold(self._h, ptr(bold), n)
        return bold.reshape(-1, self._n_voxels) if self._n_voxels else bold

    def set_hemodynamics(self, params: HemoParams | None = None, baseline_hz: float = 1.0,
                         sample_every: int = 1, state: np.ndarray | None = None) -> None:
        """Device BOLD-proxy readout for every following advance: the
        assimilation caller's window_bold (assim.cpp:51-71) per voxel, sampled
        like bold_from_drive (hemo.cpp:49-62); `state` seeds the per-voxel
        HemoState (default: rest) and then carries across advances."""
        p = params or HemoParams()
        st = None
        if state is not None:
            st = np.ascontiguousarray(state, HEMO_STATE_DTYPE)
            if st.size != self._n_voxels:
                raise ConfigError("hemodynamic state size does not match the voxel count")
        rc = self._lib.vxb_set_hemodynamics(self._h, C.byref(p._c()), baseline_hz, sample_every,
                                            ptr(st))
        if rc != 0:
            self._err(rc)
        self._hemo_every = sample_every

    def hemo_state(self) -> np.ndarray:
        """Per-voxel HemoState after the last advance (HEMO_STATE_DTYPE)."""
        out = np.zeros(self._n_voxels, HEMO_STATE_DTYPE)
        rc = self._lib.vxb_hemo_get_state(self._h, ptr(out), out.size)
        if rc != 0:
            self._err(rc)
        return out

    def set_conductances(self, unit: int, receptor: int, values) -> None:
        v = np.ascontiguousarray(values, dtype=np.float32)
        # (per-window hot call of the assimilation caller: from_buffer is ~2x
        # cheaper than ndarray.ctypes for the address of a writable buffer)
        try:
            addr = C.addressof(C.c_char.from_buffer(v)) if v.size else None
        except (TypeError, ValueError):
            addr = ptr(v)
        rc = self._lib.vxb_set_conductances(self._h, unit, receptor, addr, v.size)
        if rc != 0:
            self._err(rc)

    def set_conductances_batch(self, items) -> int:
        """set_conductances for many (unit, receptor, values) in one call:
        the result and errors of calling it item by item (staging stops at
        the first failing item), validated and copied on several host cores
        (vxb_set_conductances_batch).  `items` is a list or a prebuilt
        ConductanceBatch (whose buffers may be refilled between calls)."""
        b = items if isinstance(items, ConductanceBatch) else ConductanceBatch(items)
        failed = C.c_uint32(0)
        rc = self._lib.vxb_set_conductances_batch(self._h, b.n, b.units_p, b.recs_p, b.ptrs,
                                                  b.counts_p, C.byref(failed))
        if rc != 0:
            self.failed_index = int(failed.value)
            self._err(rc)
        return b.n

    def membrane_snapshot(self, worker: int) -> np.ndarray:
        n = int(self._lib.vxb_worker_neurons(self._h, worker)) if worker < self.workers else 0
        out = np.zeros(max(n, 1), np.float32)
        rc = self._lib.vxb_membrane_snapshot(self._h, worker, ptr(out), out.size)
        if rc != 0:
            self._err(rc)
        return out[:n]

    @property
    def workers(self) -> int:
        return int(self._lib.vxb_workers(self._h))

    def crossing_matrix(self) -> np.ndarray:
        """BuiltNetwork::crossing (netgen.cpp:331-355): synapses per (source
        worker, target worker) of the tables this instance holds."""
        w = self.workers
        out = np.zeros((w, w), np.uint64)
        rc = self._lib.vxb_crossing_matrix(self._h, ptr(out), out.size)
        if rc != 0:
            self._err(rc)
        return out

    def schedule_info(self) -> dict:
        """The delivery schedule the engine chose (and any tuning knob applied
        from the environment under VXB_TUNING=1), for benchmark records."""
        import json
        buf = C.create_string_buffer(4096)
        rc = self._lib.vxb_schedule_info(self._h, buf, len(buf))
        if rc != 0:
            self._err(rc)
        return json.loads(buf.value.decode())


def advance_members(members: Sequence["SimInstance"], steps: int) -> List[RunResult]:
    """Advance ensemble members of one donor together (vxb_advance_members):
    concurrently on shares of the SMs where their path allows it, else one
    after another; returns each member's RunResult."""
    if not members:
        return []
    lib = members[0]._lib
    hs = (C.c_void_p * len(members))(*[m._h.value if isinstance(m._h, C.c_void_p) else m._h
                                       for m in members])
    rc = lib.vxb_advance_members(hs, len(members), steps)
    if rc != 0:
        for m in members:
            msg = lib.vxb_last_error(m._h).decode()
            if msg:
                _raise(rc, msg)
        _raise(rc, "advance_members failed")
    return [m.result() for m in members]


def run_simulation(tables: NetworkTables, options: SimOptions) -> RunResult:
    """voxsim::run_simulation (engine.hpp:92-93)."""
    with SimInstance(tables, options) as sim:
        return sim.advance(options.steps)
