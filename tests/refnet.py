"""Test-side bindings of the CPU checkers in oracle/_ref/ (test infrastructure).

* RefNet / RefSim wrap libvoxsim_ref.so: the UNMODIFIED reference engine built
  from /root/reference/proj/src by oracle/Makefile, driven through its own API
  (pipeline.cpp build_network / emit_tables, engine.cpp SimInstance).
* OracleSim wraps libvoxsim_oracle.so: the plain-C restatement
  oracle/voxsim_oracle.c.

Both consume / produce the vxb.h table layout so the CUDA engine can be run
on byte-identical inputs.  Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from paper_2308_01241_b200 import _abi
from paper_2308_01241_b200._abi import (NEURON_DTYPE, RASTER_DTYPE, SYN_DTYPE, TIMINGS_DTYPE,
                                        UNIT_DTYPE, ptr)
from paper_2308_01241_b200.engine import (ConfigError, NetworkTables, SimError, SimOptions,
                                          WorkerTable)

ROOT = Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libvoxsim_ref.so"
ORACLE_SO = ROOT / "oracle" / "_ref" / "libvoxsim_oracle.so"

_ref = None
_orc = None


def ref_lib():
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle`")
        L = C.CDLL(str(REF_SO))
        P, u64, u32, u16 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint16
        sig = {
            "ref_build": (P, [C.c_char_p, C.c_int, C.c_char_p, C.c_int]),
            "ref_free": (None, [P]),
            "ref_save_tables": (C.c_int, [P, C.c_char_p, C.c_char_p, C.c_int]),
            "ref_load_net": (P, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]),
            "ref_build_seconds": (C.c_double, [P]),
            "ref_seed": (u64, [P]),
            "ref_n_workers": (u32, [P]),
            "ref_n_units": (u32, [P]),
            "ref_n_voxels": (u32, [P]),
            "ref_total_neurons": (u64, [P]),
            "ref_synapse_count": (u64, [P]),
            "ref_crossing": (C.c_int, [P, P, u32]),
            "ref_worker_n": (u32, [P, u32]),
            "ref_worker_nsyn": (u64, [P, u32]),
            "ref_units": (None, [P, P, P, P]),
            "ref_worker_neurons": (None, [P, u32, P]),
            "ref_worker_synapses": (None, [P, u32, P, P]),
            "ref_sim_create": (P, [P, C.c_char_p, C.c_char_p, C.c_int]),
            "ref_sim_free": (None, [P]),
            "ref_sim_advance": (C.c_int, [P, u32, C.c_char_p, C.c_int]),
            "ref_sim_advance_seconds": (C.c_double, [P]),
            "ref_sim_current_step": (u32, [P]),
            "ref_res_total_spikes": (u64, [P]),
            "ref_res_steps_done": (u32, [P]),
            "ref_res_raster_size": (u64, [P]),
            "ref_res_raster": (None, [P, P]),
            "ref_res_rates": (None, [P, P]),
            "ref_res_n_probes": (u32, [P]),
            "ref_res_probes": (None, [P, P, P]),
            "ref_res_flops": (None, [P, P]),
            "ref_res_timings_size": (u64, [P]),
            "ref_res_timings": (None, [P, P]),
            "ref_sim_set_conductances": (C.c_int, [P, u32, C.c_int, P, u32, C.c_char_p, C.c_int]),
            "ref_sim_snapshot": (C.c_int, [P, u16, P, u32, C.c_char_p, C.c_int]),
            "ref_splitmix64": (u64, [u64]),
            "ref_mix_key2": (u64, [u64, u64]),
            "ref_mix_key3": (u64, [u64, u64, u64]),
            "ref_stream_word": (u64, [u64, u64]),
            "ref_stream_u01": (C.c_double, [u64, u64]),
            "ref_stream_normal": (C.c_double, [u64, u64]),
            "ref_stream_below": (u64, [u64, u64, u64]),
            "ref_quantize_weight": (C.c_int32, [C.c_double]),
            "ref_dequantize_weight": (C.c_float, [C.c_int64]),
            "ref_gating_kernel": (C.c_float, [C.c_float] * 5),
            "ref_membrane_kernel": (C.c_float, [C.c_float] * 6),
            "ref_current_kernel": (C.c_float, [C.c_float, P, P, P]),
            "ref_ou_kernel": (C.c_float, [C.c_float] * 6),
            "ref_ou_xi": (C.c_float, [u64, u64, u64]),
            "ref_bold_from_drive": (C.c_int, [P, P, u32, C.c_double, u32, P, P, C.c_char_p,
                                              C.c_int]),
            "ref_window_bold": (C.c_int, [P, P, u32, u32, P, u32, P, C.c_double, C.c_double,
                                          u32, P, P, C.c_char_p, C.c_int]),
            "ref_unit_pop": (None, [P, u32, P, P]),
            "ref_assimilate": (C.c_int, [P, P, u32, u32, P, P, P, u32, P, P, P, P, C.c_char_p,
                                         C.c_int]),
            "ref_forward_bold": (C.c_int, [P, P, P, P, u32, u32, P, P, C.c_char_p, C.c_int]),
            "ref_ensrf": (C.c_int, [P, P, P, u32, u32, u32, C.c_double, C.c_double, C.c_double,
                                    C.c_char_p, C.c_int]),
            "ref_sample_conductances": (None, [u64, u64, u32, C.c_int, C.c_double, C.c_double,
                                               u32, P]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _ref = L
    return _ref


def oracle_lib():
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(str(ORACLE_SO))
        P, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32
        sig = {
            "vxo_create": (P, [C.POINTER(_abi.Network), C.POINTER(_abi.Options), C.c_char_p,
                               C.c_int, C.POINTER(C.c_int)]),
            "vxo_destroy": (None, [P]),
            "vxo_last_error": (C.c_char_p, [P]),
            "vxo_advance": (C.c_int, [P, u32]),
            "vxo_current_step": (u32, [P]),
            "vxo_total_spikes": (u64, [P]),
            "vxo_raster_size": (u64, [P]),
            "vxo_raster": (None, [P, P]),
            "vxo_rates": (None, [P, P]),
            "vxo_probes": (None, [P, P, P]),
            "vxo_flops": (None, [P, C.POINTER(_abi.Flops)]),
            "vxo_worker_n": (u32, [P, u32]),
            "vxo_snapshot": (None, [P, u32, P]),
            "vxo_splitmix64": (u64, [u64]),
            "vxo_mix_key": (u64, [u64, u64]),
            "vxo_stream_word": (u64, [u64, u64]),
            "vxo_stream_u01": (C.c_double, [u64, u64]),
            "vxo_stream_normal": (C.c_double, [u64, u64]),
            "vxo_stream_below": (u64, [u64, u64, u64]),
            "vxo_ou_xi": (C.c_float, [u64, u64, u64]),
            "vxo_quantize_weight": (C.c_int32, [C.c_double]),
            "vxo_dequantize_weight": (C.c_float, [C.c_int64]),
            "vxo_gating_kernel": (C.c_float, [C.c_float] * 5),
            "vxo_current_kernel": (C.c_float, [C.c_float, P, P, P]),
            "vxo_membrane_kernel": (C.c_float, [C.c_float] * 6),
            "vxo_ou_kernel": (C.c_float, [C.c_float] * 6),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _orc = L
    return _orc


def _raise(rc: int, msg: str):
    if rc == 2:
        raise ConfigError(msg)
    if rc == 3:
        raise SimError(msg)
    raise RuntimeError(msg)


def _strip(msg: str) -> str:
    for p in ("ConfigError: ", "SimError: ", "Error: "):
        if msg.startswith(p):
            return msg[len(p):]
    return msg


# --------------------------------------------------------------- networks
def make_config(*, seed=1, voxels=1, npv=100, k_in=10, rho=0.0, kind=None, dt_ms=1.0,
                steps=100, workers=1, partition="sequential", ou_mean=None, ou_sigma=None,
                g_location=None, region="subcortex", extra_region=None, connectome=None):
    """RunConfig JSON (config.hpp:40-60) for the reference pipeline."""
    if kind is None:
        kind = "single" if voxels == 1 else "ring"
    reg = {"k_in": k_in, "rho": rho}
    if ou_mean is not None:
        reg["ou_mean"] = ou_mean
    if ou_sigma is not None:
        reg["ou_sigma"] = ou_sigma
    if g_location is not None:
        reg["g_location"] = list(g_location)
    if extra_region:
        reg.update(extra_region)
    con = {"kind": kind, "voxels": voxels, "neurons_per_voxel": npv}
    if connectome:
        con.update(connectome)
    if kind == "single":
        con.pop("voxels")
    return {"seed": seed, "dt_ms": dt_ms, "steps": steps, "workers": workers,
            "scheduler": "loopback", "connectome": con,
            "partition": {"method": partition}, "regions": {region: reg}}


class RefNet:
    """A network built by the reference pipeline, exported as NetworkTables."""

    def __init__(self, cfg: dict, even_workers: int = 0, tables_dir: str | None = None):
        L = ref_lib()
        err = C.create_string_buffer(1024)
        if tables_dir is not None:
            self._h = L.ref_load_net(json.dumps(cfg).encode(), str(tables_dir).encode(), err,
                                     1024)
        else:
            self._h = L.ref_build(json.dumps(cfg).encode(), even_workers, err, 1024)
        if not self._h:
            m = err.value.decode()
            _raise(2 if m.startswith("ConfigError") else 3, _strip(m))
        self.cfg = cfg
        self.build_seconds = L.ref_build_seconds(self._h)
        self.tables = self._export()

    def __del__(self):
        try:
            if self._h:
                ref_lib().ref_free(self._h)
        except Exception:
            pass

    def _export(self) -> NetworkTables:
        L, h = ref_lib(), self._h
        nu, nw = L.ref_n_units(h), L.ref_n_workers(h)
        units = np.zeros(nu, UNIT_DTYPE)
        uw = np.zeros(nu, np.uint16)
        ulb = np.zeros(nu, np.uint32)
        L.ref_units(h, ptr(units), ptr(uw), ptr(ulb))
        seed = L.ref_seed(h)
        workers = []
        for w in range(nw):
            n, ns = L.ref_worker_n(h, w), L.ref_worker_nsyn(h, w)
            neurons = np.zeros(n, NEURON_DTYPE)
            syn = np.zeros(ns, SYN_DTYPE)
            rb = np.zeros(n + 1, np.uint64)
            if n:
                L.ref_worker_neurons(h, w, ptr(neurons))
            L.ref_worker_synapses(h, w, ptr(syn) if ns else None, ptr(rb))
            workers.append(WorkerTable(w, nw, seed, neurons, syn, rb))
        return NetworkTables(workers, uw, ulb, units, L.ref_n_voxels(h))

    @property
    def total_neurons(self) -> int:
        return int(ref_lib().ref_total_neurons(self._h))

    def crossing(self) -> np.ndarray:
        """BuiltNetwork::crossing, [src worker][dst worker] synapse counts."""
        w = len(self.tables.workers)
        out = np.zeros((w, w), np.uint64)
        if not ref_lib().ref_crossing(self._h, ptr(out), w):
            raise RuntimeError("network not built through build_network")
        return out

    def save_tables(self, directory) -> None:
        err = C.create_string_buffer(1024)
        rc = ref_lib().ref_save_tables(self._h, str(directory).encode(), err, 1024)
        if rc:
            _raise(rc, _strip(err.value.decode()))


@dataclass
class CpuResult:
    raster: np.ndarray
    rates: np.ndarray
    probe_v: np.ndarray
    probe_i: np.ndarray
    flops: dict
    total_spikes: int
    seconds: float = 0.0


def _opts_json(o: SimOptions, scheduler: str) -> str:
    return json.dumps({
        "steps": o.steps, "dt_ms": o.dt_ms, "scheduler": scheduler, "transport": o.transport,
        "workers_per_node": o.workers_per_node, "recv_timeout_ms": o.recv_timeout_ms,
        "record_raster": bool(o.record_raster), "record_timings": bool(o.record_timings),
        "probe_gids": [int(g) for g in o.probe_gids],
        "injections": [[i.from_step, i.to_step, i.voxel, i.current_pa] for i in o.injections],
        "forced_spikes": [[f.step, f.gid] for f in o.forced_spikes],
    })


class RefSim:
    """The reference voxsim::SimInstance on a RefNet (CPU)."""

    def __init__(self, net: RefNet, opt: SimOptions, scheduler: str = "loopback"):
        L = ref_lib()
        err = C.create_string_buffer(1024)
        self._net = net
        self._opt = opt
        self._h = L.ref_sim_create(net._h, _opts_json(opt, scheduler).encode(), err, 1024)
        if not self._h:
            m = err.value.decode()
            _raise(2 if m.startswith("ConfigError") else 3, _strip(m))

    def __del__(self):
        try:
            if self._h:
                ref_lib().ref_sim_free(self._h)
        except Exception:
            pass

    def advance(self, steps: int) -> CpuResult:
        L, h = ref_lib(), self._h
        err = C.create_string_buffer(1024)
        rc = L.ref_sim_advance(h, steps, err, 1024)
        if rc:
            _raise(rc, _strip(err.value.decode()))
        nr = L.ref_res_raster_size(h)
        raster = np.zeros(nr, RASTER_DTYPE)
        if nr:
            L.ref_res_raster(h, ptr(raster))
        nu = L.ref_n_units(self._net._h)
        rates = np.zeros((nu, steps), np.uint32)
        if rates.size:
            L.ref_res_rates(h, ptr(rates))
        npb = L.ref_res_n_probes(h)
        pv = np.zeros((npb, steps), np.float32)
        pi = np.zeros((npb, steps), np.float32)
        if pv.size:
            L.ref_res_probes(h, ptr(pv), ptr(pi))
        fl = np.zeros(5, np.uint64)
        L.ref_res_flops(h, ptr(fl))
        flops = dict(zip(("membrane", "gating_inner", "gating_outer", "gating_decay",
                          "current"), (int(x) for x in fl)))
        return CpuResult(raster, rates, pv, pi, flops, int(L.ref_res_total_spikes(h)),
                         L.ref_sim_advance_seconds(h))

    def timings(self) -> np.ndarray:
        L, h = ref_lib(), self._h
        n = L.ref_res_timings_size(h)
        t = np.zeros(n, TIMINGS_DTYPE)
        if n:
            L.ref_res_timings(h, ptr(t))
        return t

    def current_step(self) -> int:
        return int(ref_lib().ref_sim_current_step(self._h))

    def membrane_snapshot(self, worker: int) -> np.ndarray:
        n = self._net.tables.workers[worker].neurons.shape[0] if worker < len(
            self._net.tables.workers) else 0
        out = np.zeros(max(n, 1), np.float32)
        err = C.create_string_buffer(1024)
        rc = ref_lib().ref_sim_snapshot(self._h, worker, ptr(out), out.size, err, 1024)
        if rc:
            _raise(rc, _strip(err.value.decode()))
        return out[:n]

    def set_conductances(self, unit, receptor, values):
        v = np.ascontiguousarray(values, np.float32)
        err = C.create_string_buffer(1024)
        rc = ref_lib().ref_sim_set_conductances(self._h, unit, receptor, ptr(v), v.size, err,
                                                1024)
        if rc:
            _raise(rc, _strip(err.value.decode()))


class OracleSim:
    """The C restatement oracle/voxsim_oracle.c on the same tables (CPU)."""

    def __init__(self, tables: NetworkTables, opt: SimOptions):
        L = oracle_lib()
        self._tables = tables
        net, self._keep_net = tables._descriptor()
        o, self._keep_opt = opt._descriptor()
        self._opt = opt
        err = C.create_string_buffer(1024)
        rc = C.c_int(0)
        self._h = L.vxo_create(C.byref(net), C.byref(o), err, 1024, C.byref(rc))
        if not self._h:
            _raise(rc.value, _strip(err.value.decode()))

    def __del__(self):
        try:
            if self._h:
                oracle_lib().vxo_destroy(self._h)
        except Exception:
            pass

    def advance(self, steps: int) -> CpuResult:
        L, h = oracle_lib(), self._h
        rc = L.vxo_advance(h, steps)
        if rc:
            _raise(rc, _strip(L.vxo_last_error(h).decode()))
        nr = L.vxo_raster_size(h)
        raster = np.zeros(nr, RASTER_DTYPE)
        if nr:
            L.vxo_raster(h, ptr(raster))
        nu = self._tables.units.shape[0]
        rates = np.zeros((nu, steps), np.uint32)
        if rates.size:
            L.vxo_rates(h, ptr(rates))
        npb = len(self._opt.probe_gids)
        pv = np.zeros((npb, steps), np.float32)
        pi = np.zeros((npb, steps), np.float32)
        if pv.size:
            L.vxo_probes(h, ptr(pv), ptr(pi))
        fl = _abi.Flops()
        L.vxo_flops(h, C.byref(fl))
        flops = {n: int(getattr(fl, n)) for n, _ in _abi.Flops._fields_}
        return CpuResult(raster, rates, pv, pi, flops, int(L.vxo_total_spikes(h)))

    def membrane_snapshot(self, worker: int) -> np.ndarray:
        L = oracle_lib()
        n = L.vxo_worker_n(self._h, worker)
        out = np.zeros(max(n, 1), np.float32)
        L.vxo_snapshot(self._h, worker, ptr(out))
        return out[:n]


def raster_set(raster: np.ndarray):
    """Multiset of (step, gid), as test_engine.cpp:98-103."""
    return sorted(zip(raster["step"].tolist(), raster["gid"].tolist()))


# ---------------------------------------------------------- hemodynamics
def _hemo_p(params):
    return np.array([params.kappa, params.gamma, params.tau, params.alpha, params.e0,
                     params.v0], np.float64)


def ref_bold_from_drive(params, z, dt_s, sample_every, state=None):
    """The reference's bold_from_drive (hemo.cpp:49-62); state = [s, f, v, q]
    (float64[4], updated in place) or rest."""
    L = ref_lib()
    z = np.ascontiguousarray(z, np.float64)
    st = np.array([0.0, 1.0, 1.0, 1.0]) if state is None else state
    out = np.zeros(len(z) // max(1, sample_every), np.float64)
    err = C.create_string_buffer(1024)
    rc = L.ref_bold_from_drive(ptr(_hemo_p(params)), ptr(z), len(z), dt_s, sample_every,
                               ptr(st), ptr(out), err, 1024)
    if rc:
        _raise(rc, _strip(err.value.decode()))
    return out


def ref_window_bold(params, counts, unit_voxel, vox_n, dt_s, baseline_hz, sample_every,
                    states):
    """window_bold (assim.cpp:51-71) with bold_from_drive sampling, around the
    reference's step_hemodynamics / bold_signal; states float64[voxels][4] in/out."""
    L = ref_lib()
    counts = np.ascontiguousarray(counts, np.uint32)
    nu, steps = counts.shape
    uv = np.ascontiguousarray(unit_voxel, np.uint32)
    vn = np.ascontiguousarray(vox_n, np.uint64)
    out = np.zeros((steps // sample_every, len(vn)), np.float64)
    err = C.create_string_buffer(1024)
    rc = L.ref_window_bold(ptr(_hemo_p(params)), ptr(counts), nu, steps, ptr(uv), len(vn),
                           ptr(vn), dt_s, baseline_hz, sample_every, ptr(states), ptr(out),
                           err, 1024)
    if rc:
        _raise(rc, _strip(err.value.decode()))
    return out


# ---------------------------------------------------------- assimilation
def _assim_args(opts):
    h = opts.hemo
    d = np.array([opts.dt_ms, opts.obs_noise_sd, opts.inflation, opts.min_spread, opts.prior_sd,
                  opts.baseline_hz, opts.divergence_factor, h.kappa, h.gamma, h.tau, h.alpha,
                  h.e0, h.v0], np.float64)
    iv = np.array([opts.members, opts.windows, opts.window_steps, opts.divergence_patience,
                   opts.seed], np.int64)
    tg = np.array([[t.unit, t.receptor] for t in opts.targets], np.uint32).reshape(-1)
    return d, iv, tg


def ref_unit_pop(net, unit):
    """(g_location[4], g_scale[4]) of the unit's population (layout.pop_of_unit)."""
    gl, gs = np.zeros(4), np.zeros(4)
    ref_lib().ref_unit_pop(net._h, unit, ptr(gl), ptr(gs))
    return gl, gs


def ref_assimilate(net, observed, opts):
    """The reference's assimilate (assim.cpp:181-299) on a RefNet."""
    L = ref_lib()
    obs = np.ascontiguousarray(observed, np.float64)
    d, iv, tg = _assim_args(opts)
    nt = len(opts.targets)
    stats = np.zeros((obs.shape[0], 4 + nt))
    fin = np.zeros(2 * nt)
    ns, div = C.c_uint32(0), C.c_int(0)
    err = C.create_string_buffer(1024)
    rc = L.ref_assimilate(net._h, ptr(obs), obs.shape[0], obs.shape[1], ptr(d), ptr(iv), ptr(tg),
                          nt, ptr(stats), C.byref(ns), ptr(fin), C.byref(div), err, 1024)
    if rc:
        _raise(rc, _strip(err.value.decode()))
    return stats[:ns.value], fin[:nt], fin[nt:], div.value


def ref_forward_bold(net, opts, windows, true_params=None):
    L = ref_lib()
    d, iv, tg = _assim_args(opts)
    tp = None if true_params is None else np.ascontiguousarray(true_params, np.float64)
    out = np.zeros((windows, net.tables.n_voxels))
    err = C.create_string_buffer(1024)
    rc = L.ref_forward_bold(net._h, ptr(d), ptr(iv), ptr(tg), len(opts.targets), windows,
                            ptr(tp), ptr(out), err, 1024)
    if rc:
        _raise(rc, _strip(err.value.decode()))
    return out


def ref_ensrf(ensemble, forecasts, obs, obs_var, inflation, min_spread):
    """EnsrfUpdate::apply (assim.cpp:108-179); returns the updated ensemble."""
    e = np.ascontiguousarray(ensemble, np.float64).copy()
    f = np.ascontiguousarray(forecasts, np.float64)
    o = np.ascontiguousarray(obs, np.float64)
    err = C.create_string_buffer(1024)
    rc = ref_lib().ref_ensrf(ptr(e), ptr(f), ptr(o), e.shape[0], e.shape[1], o.size, obs_var,
                             inflation, min_spread, err, 1024)
    if rc:
        _raise(rc, _strip(err.value.decode()))
    return e


def ref_sample_conductances(seed, salt, unit, receptor, location, scale, count):
    out = np.zeros(count, np.float32)
    ref_lib().ref_sample_conductances(seed, salt, unit, receptor, location, scale, count,
                                      ptr(out))
    return out
