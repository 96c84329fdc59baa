"""Network build for the B200 engine: RunConfig -> connectome -> layout ->
partition -> vxb_netspec, then on-device synapse generation.

Mirrors the reference pipeline (/root/reference/proj/src/pipeline.cpp:49-125)
step by step so a config produces the same network the reference builds:

  parse/validate       config.hpp:40-60, config.cpp:133-176 (same JSON schema)
  build_connectome     pipeline.cpp:49-73, connectome.cpp:68-227
  build_layout         pipeline.cpp:75-96, layout.cpp:28-117, 146-186
  partition            partition.cpp:44-352 (unit graph, greedy, sequential,
                       exact, file) + an "even" helper (test_engine.cpp:40-47)
  sample/emit          on the device: vxb_create_generated (include/vxb.h)

Host work here is O(voxels^2 + units^2); the O(neurons * K) synapse draws run
on the GPU.  Random quantities use the reference's counter streams; the libm
calls (exp/log/cos/pow) are the same glibc functions the reference calls.
"""
from __future__ import annotations

import copy
import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import _abi
from ._abi import NEURON_DTYPE, SYN_DTYPE, UNIT_DTYPE, ptr
from .engine import ConfigError, NetworkTables, SimError, SimInstance, SimOptions, WorkerTable

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
RNG_CONDUCTANCE = 7  # rng.hpp:17-28 stream tag


# ---------------------------------------------------------------- rng.hpp
def splitmix64(x: int) -> int:
    x = (x + GOLDEN) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def mix_key(a: int, *rest: int) -> int:
    for b in rest:
        a = splitmix64(a ^ ((b + GOLDEN + ((a << 6) & MASK64) + (a >> 2)) & MASK64))
    return a


def stream_word(base: int, k: int) -> int:
    return splitmix64((base + k * GOLDEN) & MASK64)


def stream_u01(base: int, k: int) -> float:
    return float(stream_word(base, k) >> 11) * 2.0 ** -53


def stream_normal(base: int, k: int) -> float:
    u1 = 1.0 - stream_u01(base, 2 * k)
    u2 = stream_u01(base, 2 * k + 1)
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586476925286766559 * u2)


def stream_normal_array(base: int, count: int) -> np.ndarray:
    """stream_normal(base, k) for k in [0, count), vectorised (rng.hpp:58-67).
    The integer stream is exact; numpy's log/cos may differ from glibc's in
    the last ulp, so this feeds workloads (bench inputs), never parity."""
    k = np.arange(count, dtype=np.uint64)

    def u01(j):
        with np.errstate(over="ignore"):
            x = np.uint64(base) + j * np.uint64(GOLDEN) + np.uint64(GOLDEN)
            x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
        return (x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    u1 = 1.0 - u01(2 * k)
    u2 = u01(2 * k + np.uint64(1))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586476925286766559 * u2)


def sample_conductances(seed: int, salt: int, unit: int, receptor: int, location: float,
                        scale: float, count: int) -> np.ndarray:
    """netgen.cpp:318-329 (vectorised; see stream_normal_array for the ulp note).
    salt 0 draws the tables' initial values; assim.cpp:98-103 uses
    mix_key(member + 1, window + 1) per assimilation window."""
    base = mix_key(mix_key(seed, RNG_CONDUCTANCE, salt), unit, receptor)
    return np.exp(location + scale * stream_normal_array(base, count)).astype(np.float32)


def sample_conductances_exact(seed: int, salt: int, unit: int, receptor: int,
                              location: float, scale: float, count: int) -> np.ndarray:
    """sample_conductances (netgen.cpp:318-329) with glibc's log/cos/exp
    (Python's math): the reference's values bit for bit.  Scalar — for the
    per-window conductances of the assimilation loop (assim.py)."""
    base = mix_key(mix_key(seed, RNG_CONDUCTANCE, salt), unit, receptor)
    out = np.empty(count, np.float32)
    for i in range(count):
        out[i] = math.exp(location + scale * stream_normal(base, i))
    return out


def stream_below(base: int, k: int, n: int) -> int:
    return stream_word(base, k) % n


def f32(x: float) -> float:
    return float(np.float32(x))


def llround(x: float) -> int:
    """std::llround: nearest, halves away from zero."""
    if x < 0:
        return -llround(-x)
    r = math.floor(x)
    return int(r) + (1 if x - r >= 0.5 else 0)


REGIONS = ["cortex", "subcortex", "brainstem", "cerebellum"]
REGION_DEFAULTS = {  # layout.cpp:28-36
    "cortex": (1000, 2.0 / 7.0),
    "subcortex": (1000, 6.0 / 25.0),
    "brainstem": (100, 14.0 / 25.0),
    "cerebellum": (100, 16.0 / 125.0),
}


# ------------------------------------------------------------- population
@dataclass
class NeuronParams:  # model.hpp:30-44
    capacitance: float = 250.0
    g_leak: float = 25.0
    e_leak: float = -65.0
    v_threshold: float = -50.0
    v_reset: float = -65.0
    refractory_steps: int = 2
    e_rev: List[float] = field(default_factory=lambda: [0.0, 0.0, -70.0, -70.0])
    tau: List[float] = field(default_factory=lambda: [4.0, 100.0, 10.0, 200.0])
    omega: List[float] = field(default_factory=lambda: [0.5, 0.05, 0.5, 0.05])
    g: List[float] = field(default_factory=lambda: [1.0, 0.15, 4.0, 0.5])

    def validate(self, dt_ms: float):  # model.cpp:7-26 (float compares)
        if not f32(self.capacitance) > 0:
            raise ConfigError("neuron params: capacitance must be > 0")
        if f32(self.g_leak) < 0:
            raise ConfigError("neuron params: leak conductance must be >= 0")
        if not f32(self.v_reset) < f32(self.v_threshold):
            raise ConfigError("neuron params: V_reset must be below V_th")
        for u in range(4):
            if not f32(self.tau[u]) > 0:
                raise ConfigError("neuron params: receptor tau must be > 0")
            if not f32(dt_ms) < f32(self.tau[u]):
                raise ConfigError("neuron params: dt must be below every receptor tau "
                                  "(explicit Euler)")
            if f32(self.g[u]) < 0 or f32(self.omega[u]) < 0:
                raise ConfigError("neuron params: receptor conductance and jump weights "
                                  "must be >= 0")
        if f32(self.e_rev[0]) <= f32(self.v_threshold) or f32(self.e_rev[1]) <= f32(self.v_threshold):
            raise ConfigError("neuron params: excitatory reversals must lie above V_th")
        if f32(self.e_rev[2]) >= f32(self.e_leak) or f32(self.e_rev[3]) >= f32(self.e_leak):
            raise ConfigError("neuron params: inhibitory reversals must lie below E_L")


@dataclass
class PopulationSpec:  # layout.hpp:17-38
    label: str = ""
    excitatory: bool = True
    fraction: float = 0.0
    layer: int = -1
    neuron: NeuronParams = field(default_factory=NeuronParams)
    ou_mean: float = 225.0
    ou_sigma: float = 120.0
    ou_tau: float = 10.0
    g_location: List[float] = field(default_factory=lambda: [
        0.0, -1.8971199848858813, 2.0794415416798357, -0.6931471805599453])
    g_scale: List[float] = field(default_factory=lambda: [0.2, 0.2, 0.2, 0.2])
    weight_mean: List[float] = field(default_factory=lambda: [1.0, 1.0, 1.0, 1.0])
    weight_spread: List[float] = field(default_factory=lambda: [0.2, 0.2, 0.2, 0.2])
    dual_receptor: bool = True
    split_ratio: float = 0.5


@dataclass
class VoxelSpec:  # layout.hpp:40-49
    id: int
    region: str
    neurons: int
    k_in: int
    rho: float
    populations: List[PopulationSpec]

    def validate(self):  # layout.cpp:38-58
        if self.neurons == 0:
            raise ConfigError("voxel with zero neurons")
        if self.rho < 0.0 or self.rho > 1.0:
            raise ConfigError("rho outside [0, 1]")
        if not self.populations:
            raise ConfigError("voxel with no populations")
        total = 0.0
        for p in self.populations:
            if p.fraction < 0.0:
                raise ConfigError("negative population fraction")
            total += p.fraction
            p.neuron.validate(1.0)
            for r in range(4):
                if p.g_scale[r] < 0.0:
                    raise ConfigError("negative conductance scale")
                if p.weight_spread[r] < 0.0:
                    raise ConfigError("negative weight spread")
            if p.split_ratio < 0.0 or p.split_ratio > 1.0:
                raise ConfigError("split_ratio outside [0, 1]")
            if f32(p.ou_sigma) < 0.0 or f32(p.ou_tau) <= 0.0:
                raise ConfigError("bad noise parameters")
        if abs(total - 1.0) > 1e-9:
            raise ConfigError("population fractions must sum to 1")


@dataclass
class Unit:  # layout.hpp:53-60
    id: int
    voxel: int
    pop: int
    excitatory: bool
    neurons: int
    gid_base: int


@dataclass
class Layout:  # NetworkLayout (layout.hpp:64-83)
    voxels: List[VoxelSpec]
    units: List[Unit]
    voxel_unit_base: List[int]
    total_neurons: int

    def unit_of_gid(self, gid: int) -> Unit:
        if gid >= self.total_neurons:
            raise SimError("gid out of range")
        lo, hi = 0, len(self.units)
        while lo < hi:
            mid = (lo + hi) // 2
            if gid < self.units[mid].gid_base:
                hi = mid
            else:
                lo = mid + 1
        i = lo - 1
        while self.units[i].neurons == 0:
            i -= 1
        return self.units[i]

    def excitatory_count(self, v: int) -> int:
        return sum(u.neurons for u in self.units[self.voxel_unit_base[v]:self.voxel_unit_base[v + 1]]
                   if u.excitatory)

    def pop_of_unit(self, u: int) -> PopulationSpec:
        x = self.units[u]
        return self.voxels[x.voxel].populations[x.pop]


def split_counts(n: int, pops: List[PopulationSpec]) -> List[int]:  # layout.cpp:63-83
    k = len(pops)
    counts, rem, assigned = [0] * k, [], 0
    for i, p in enumerate(pops):
        exact = p.fraction * n
        counts[i] = int(exact)
        assigned += counts[i]
        rem.append((exact - counts[i], i))
    rem.sort(key=lambda t: -t[0])  # stable: ties keep lower index first
    j = 0
    while assigned < n:
        counts[rem[j % k][1]] += 1
        assigned += 1
        j += 1
    return counts


def build_layout_from_voxels(voxels: List[VoxelSpec]) -> Layout:  # layout.cpp:85-117
    if not voxels:
        raise ConfigError("layout with zero voxels")
    voxels = sorted(voxels, key=lambda v: v.id)
    for i, v in enumerate(voxels):
        if v.id != i:
            raise ConfigError("voxel ids must be 0..V-1 without gaps")
    units, base, gid = [], [], 0
    for v in voxels:
        v.validate()
        base.append(len(units))
        for p, c in enumerate(split_counts(v.neurons, v.populations)):
            units.append(Unit(len(units), v.id, p, v.populations[p].excitatory, c, gid))
            gid += c
    base.append(len(units))
    return Layout(voxels, units, base, gid)


# ------------------------------------------------------------- connectome
@dataclass
class Connectome:  # connectome.hpp:21-36
    voxel_count: int
    edges: List[tuple]          # (src, dst, weight) sorted by (dst, src)
    region: List[str]
    neuron_count: List[int]
    gm_weight: List[float]

    def validate(self):  # connectome.cpp:13-37
        if self.voxel_count == 0:
            raise ConfigError("connectome with zero voxels")
        if not (len(self.region) == len(self.neuron_count) == len(self.gm_weight) == self.voxel_count):
            raise ConfigError("connectome metadata size mismatch")
        for v in range(self.voxel_count):
            if self.neuron_count[v] == 0:
                raise ConfigError(f"voxel {v} has zero neurons")
            if not self.gm_weight[v] >= 0.0:
                raise ConfigError(f"negative gm weight on voxel {v}")
        prev = None
        for (s, d, w) in self.edges:
            if s >= self.voxel_count or d >= self.voxel_count:
                raise ConfigError("edge endpoint out of range")
            if s == d:
                raise ConfigError(f"self-loop edge on voxel {s}")
            if not w >= 0.0:
                raise ConfigError("negative edge weight")
            if prev is not None and (d < prev[1] or (d == prev[1] and s <= prev[0])):
                raise ConfigError("edges must be sorted by (dst, src), unique")
            prev = (s, d)


def _blank(voxels, npv):
    return Connectome(voxels, [], ["subcortex"] * voxels, [npv] * voxels, [1.0] * voxels)


def _sort(g):
    g.edges.sort(key=lambda e: (e[1], e[0]))


def make_ring(voxels, npv):  # connectome.cpp:68-80
    if voxels < 3:
        raise ConfigError("ring connectome needs >= 3 voxels")
    g = _blank(voxels, npv)
    for v in range(voxels):
        g.edges.append((v, (v + voxels - 1) % voxels, 1.0))
        g.edges.append((v, (v + 1) % voxels, 1.0))
    _sort(g)
    g.validate()
    return g


def make_uniform(voxels, npv, sparsity, weight_sigma, gm_sigma, seed):  # connectome.cpp:82-114
    if voxels < 2:
        raise ConfigError("uniform connectome needs >= 2 voxels")
    if sparsity < 0.0 or sparsity > 1.0:
        raise ConfigError("sparsity outside [0, 1]")
    g = _blank(voxels, npv)
    present, weight = mix_key(seed, 8, 0), mix_key(seed, 8, 3)
    # vectorised u01 over all ordered pairs (k = s * V + d)
    k = np.arange(voxels * voxels, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = (np.uint64(present) + k * np.uint64(GOLDEN)) + np.uint64(GOLDEN)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    u = (x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    has_in = [False] * voxels
    for kk in np.nonzero(u < sparsity)[0].tolist():
        s, d = divmod(kk, voxels)
        if s == d:
            continue
        g.edges.append((s, d, math.exp(weight_sigma * stream_normal(weight, kk))))
        has_in[d] = True
    for v in range(voxels):
        if not has_in[v]:
            g.edges.append(((v + 1) % voxels, v, 1.0))
    if gm_sigma > 0.0:
        gb = mix_key(seed, 8, 1)
        g.gm_weight = [math.exp(gm_sigma * stream_normal(gb, v)) for v in range(voxels)]
    _sort(g)
    g.validate()
    return g


def make_two_block(voxels, npv, cross_weight, scramble, seed):  # connectome.cpp:116-142
    if voxels < 4:
        raise ConfigError("two_block connectome needs >= 4 voxels")
    if cross_weight < 0.0:
        raise ConfigError("negative cross_weight")
    perm = list(range(voxels))
    if scramble:
        base = mix_key(seed, 8, 2)
        for i in range(voxels - 1, 0, -1):
            j = stream_below(base, i, i + 1)
            perm[i], perm[j] = perm[j], perm[i]
    g = _blank(voxels, npv)
    half = voxels // 2
    for s in range(voxels):
        for d in range(voxels):
            if s == d:
                continue
            w = 1.0 if (s < half) == (d < half) else cross_weight
            if w > 0.0:
                g.edges.append((perm[s], perm[d], w))
    _sort(g)
    g.validate()
    return g


def make_single(npv):  # connectome.cpp:144-148
    g = _blank(1, npv)
    g.validate()
    return g


def load_connectome_text(text: str) -> Connectome:  # connectome.hpp:64-75 text format
    toks = []
    for line in text.splitlines():
        line = line.split("#", 1)[0].strip()
        if line:
            toks.append(line.split())
    it = iter(toks)
    try:
        head = next(it)
        if head[0] != "voxels":
            raise ConfigError("connectome file: expected 'voxels N'")
        n = int(head[1])
        g = Connectome(n, [], ["subcortex"] * n, [0] * n, [1.0] * n)
        for _ in range(n):
            t = next(it)
            v = int(t[0])
            if v >= n:
                raise ConfigError("connectome file: voxel id out of range")
            if t[1] not in REGIONS:
                raise ConfigError("unknown region: " + t[1])
            g.region[v] = t[1]
            g.neuron_count[v] = int(t[2])
            if len(t) > 3:
                g.gm_weight[v] = float(t[3])
        head = next(it)
        if head[0] != "edges":
            raise ConfigError("connectome file: expected 'edges M'")
        for _ in range(int(head[1])):
            t = next(it)
            g.edges.append((int(t[0]), int(t[1]), float(t[2])))
    except (StopIteration, ValueError, IndexError):
        raise ConfigError("connectome file: truncated or malformed")
    _sort(g)
    g.validate()
    return g


def save_connectome_text(g: Connectome) -> str:
    out = [f"voxels {g.voxel_count}"]
    for v in range(g.voxel_count):
        out.append(f"{v} {g.region[v]} {g.neuron_count[v]} {g.gm_weight[v]!r}")
    out.append(f"edges {len(g.edges)}")
    out += [f"{s} {d} {w!r}" for s, d, w in g.edges]
    return "\n".join(out) + "\n"


# ----------------------------------------------------------------- config
CONFIG_KEYS = {"seed", "dt_ms", "steps", "workers", "workers_per_node", "scheduler", "transport",
               "stats_window", "recv_timeout_ms", "connectome", "partition", "regions",
               "microcolumn_path", "probe_gids"}
CONNECTOME_KEYS = {"kind", "voxels", "neurons_per_voxel", "sparsity", "weight_sigma",
                   "gm_sigma", "cross_weight", "scramble", "path", "region"}
PARTITION_KEYS = {"method", "path", "alpha", "beta", "mu", "gamma", "rate_hz", "byte_model"}
REGION_KEYS = {"k_in", "rho", "ou_mean", "ou_sigma", "ou_tau", "g_location", "g_scale",
               "weight_mean", "weight_spread", "dual_receptor", "split_ratio"}


def _check_keys(d, where, allowed):  # config.cpp:18-24
    if not isinstance(d, dict):
        raise ConfigError(f"{where} must be an object")
    for k in d:
        if k not in allowed:
            raise ConfigError(f"unknown key '{k}' in {where}")


def parse_config(cfg) -> dict:
    """RunConfig (config.hpp:40-60) with defaults filled and unknown keys
    rejected at every level (config.cpp:133-176)."""
    if isinstance(cfg, str):
        cfg = json.loads(cfg)
    cfg = copy.deepcopy(cfg)
    _check_keys(cfg, "config", CONFIG_KEYS)
    out = {"seed": 1, "dt_ms": 1.0, "steps": 1000, "workers": 1, "workers_per_node": 4,
           "scheduler": "cuda", "transport": "queue", "stats_window": 800,
           "recv_timeout_ms": 30000, "microcolumn_path": "", "probe_gids": []}
    out.update({k: v for k, v in cfg.items() if k not in ("connectome", "partition", "regions")})
    con = {"kind": "ring", "voxels": 4, "neurons_per_voxel": 100, "sparsity": 0.0072,
           "weight_sigma": 0.5, "gm_sigma": 0.0, "cross_weight": 0.01, "scramble": False,
           "path": "", "region": ""}
    if "connectome" in cfg:
        _check_keys(cfg["connectome"], "connectome", CONNECTOME_KEYS)
        con.update(cfg["connectome"])
    part = {"method": "greedy", "path": "", "alpha": 1.0, "beta": 1.0, "mu": 1.0, "gamma": 0.0,
            "rate_hz": 7.0, "byte_model": "reference"}
    if "partition" in cfg:
        _check_keys(cfg["partition"], "partition", PARTITION_KEYS)
        part.update(cfg["partition"])
    if part["method"] not in ("greedy", "exact", "sequential", "file", "even"):
        raise ConfigError("unknown partition method: " + str(part["method"]))
    if part["method"] == "file" and not part["path"]:
        raise ConfigError("partition method 'file' needs a path")
    if part["byte_model"] not in BYTE_MODELS_ALL:
        raise ConfigError("unknown byte_model: " + str(part["byte_model"]))
    regions = {}
    for name, rc in cfg.get("regions", {}).items():
        if name not in REGIONS:
            raise ConfigError("unknown region: " + name)
        _check_keys(rc, f"regions.{name}", REGION_KEYS)
        for key in ("g_location", "g_scale", "weight_mean", "weight_spread"):
            if key in rc and (not isinstance(rc[key], list) or len(rc[key]) != 4):
                raise ConfigError(f"'{key}' must be an array of 4 numbers")
        regions[name] = dict(rc)
    out["connectome"], out["partition"], out["regions"] = con, part, regions
    if out["dt_ms"] <= 0:
        raise ConfigError("dt_ms must be > 0")
    if out["workers"] == 0 or out["workers"] > 64:
        raise ConfigError("workers must be in 1..64")
    return out


def build_connectome(cfg: dict) -> Connectome:  # pipeline.cpp:49-73
    c = cfg["connectome"]
    kind = c["kind"]
    if kind == "ring":
        g = make_ring(c["voxels"], c["neurons_per_voxel"])
    elif kind == "uniform":
        g = make_uniform(c["voxels"], c["neurons_per_voxel"], c["sparsity"], c["weight_sigma"],
                         c["gm_sigma"], cfg["seed"])
    elif kind == "two_block":
        g = make_two_block(c["voxels"], c["neurons_per_voxel"], c["cross_weight"], c["scramble"],
                           cfg["seed"])
    elif kind == "single":
        g = make_single(c["neurons_per_voxel"])
    elif kind == "file":
        with open(c["path"]) as f:
            g = load_connectome_text(f.read())
    else:
        raise ConfigError("unknown connectome kind: " + kind)
    if c.get("region"):
        if c["region"] not in REGIONS:
            raise ConfigError("unknown region: " + c["region"])
        g.region = [c["region"]] * g.voxel_count
    g.validate()
    return g


def load_microcolumn(path: str) -> dict:  # config.cpp:245-285
    with open(path) as f:
        j = json.load(f)
    pops = j["populations"]
    return {"labels": [p["label"] for p in pops], "fractions": [p["fraction"] for p in pops],
            "excitatory": [bool(p["excitatory"]) for p in pops],
            "layer": [p.get("layer", -1) for p in pops], "probability": j["probability"]}


def _apply_overrides(rc: dict, base: PopulationSpec, k_in: int, rho: float):
    k_in = rc.get("k_in", k_in)
    rho = rc.get("rho", rho)
    if "ou_mean" in rc:
        base.ou_mean = f32(rc["ou_mean"])
    if "ou_sigma" in rc:
        base.ou_sigma = f32(rc["ou_sigma"])
    if "ou_tau" in rc:
        base.ou_tau = f32(rc["ou_tau"])
    for key in ("g_location", "g_scale", "weight_mean", "weight_spread"):
        if key in rc:
            setattr(base, key, [float(x) for x in rc[key]])
    if "dual_receptor" in rc:
        base.dual_receptor = bool(rc["dual_receptor"])
    if "split_ratio" in rc:
        base.split_ratio = float(rc["split_ratio"])
    return k_in, rho


def build_layout(cfg: dict, g: Connectome, mc: Optional[dict]) -> Layout:  # pipeline.cpp:75-96
    voxels = []
    for v in range(g.voxel_count):
        region = g.region[v]
        k_in, rho = REGION_DEFAULTS[region]
        base = PopulationSpec()
        if region in cfg["regions"]:
            k_in, rho = _apply_overrides(cfg["regions"][region], base, k_in, rho)
        if region == "cortex":
            if not mc:
                raise ConfigError("network has cortex voxels but no micro-column file was found")
            pops = []
            for p in range(len(mc["labels"])):
                x = copy.deepcopy(base)
                x.label, x.fraction = mc["labels"][p], mc["fractions"][p]
                x.excitatory, x.layer = mc["excitatory"][p], mc["layer"][p]
                pops.append(x)
        else:  # two_population_layout (layout.cpp:146-155)
            e, i = copy.deepcopy(base), copy.deepcopy(base)
            e.label, e.excitatory, e.fraction = "E", True, 0.8
            i.label, i.excitatory, i.fraction = "I", False, 0.2
            pops = [e, i]
        voxels.append(VoxelSpec(v, region, g.neuron_count[v], k_in, rho, pops))
    return build_layout_from_voxels(voxels)


def intra_matrices(mc: Optional[dict]) -> Dict[str, List[List[float]]]:  # layout.cpp:179-186
    m = {r: [[1.0, 1.0], [1.0, 1.0]] for r in ("subcortex", "brainstem", "cerebellum")}
    m["cortex"] = mc["probability"] if mc else []
    return m


# -------------------------------------------------------------- partition
STATE_BYTES, ENTRY_BYTES, BUFFER_BYTES = 48, 16, 12  # partition.cpp:16-18

# Capacity byte models (s1 per neuron, s2 per synapse, s3 per neuron):
#  "reference" — the CPU engine's model (partition.cpp:16-18);
#  "b200"      — what this engine actually keeps in HBM per GPU: neuron state
#                V 4 + j 16 + I_ou 4 + I_syn 4 + g 16 + two pending buffers 32 +
#                destination mask 8 + spike-log slots 8 = 92 B; 12 B per synapse
#                (u32 target + packed Q16 pair); 12 B per neuron of exchange
#                receive slots (3 step slots x 4 B id).  With this model and
#                gamma = the per-GPU HBM budget, greedy/sequential place units
#                under the 180 GB of a B200.
BYTE_MODELS = {"reference": (48, 16, 12), "b200": (92, 12, 12)}
#  "b200_time" — a time model instead of bytes: femtoseconds of one step on a
#                B200 per neuron (update + noise, 38 ps: config 3 silent,
#                760 us for 20M neurons) and per synapse (3.6 ps per delivered
#                event x rate_hz x dt: config 3 at 10 Hz, 360 us for 1e8
#                events), so greedy balances the ranks' step time; the HBM
#                fit is still checked with the "b200" bytes.
TIME_MODEL_FS = (38_000, 3_600)  # per neuron-step, per delivered event
BYTE_MODELS_ALL = set(BYTE_MODELS) | {"b200_time"}
B200_HBM_BUDGET = 170e9  # bytes per GPU left for tables + state (of 183 GB)


@dataclass
class UnitGraph:  # partition.hpp:14-22
    neurons: np.ndarray
    state_bytes: np.ndarray
    table_bytes: np.ndarray
    buffer_bytes: np.ndarray
    traffic: np.ndarray  # int64 [src][dst], micro-bytes/step


def build_unit_graph(layout: Layout, g: Connectome, intra, rate_hz: float,
                     dt_ms: float, byte_model: str = "reference") -> UnitGraph:  # partition.cpp:44-138
    if rate_hz < 0.0:
        raise ConfigError("negative traffic rate")
    U = len(layout.units)
    n = np.array([u.neurons for u in layout.units], np.int64)
    kin = np.array([layout.voxels[u.voxel].k_in for u in layout.units], np.int64)
    traffic = [[0] * U for _ in range(U)]
    dt_s = dt_ms / 1000.0

    def distinct(nn, picks):
        if nn <= 0.0 or picks <= 0.0:
            return 0.0
        return nn * (1.0 - math.pow(1.0 - 1.0 / nn, picks))

    in_edges = {}
    for (s, d, w) in g.edges:
        in_edges.setdefault(d, []).append((s, w))
    for v in range(g.voxel_count):
        vx = layout.voxels[v]
        m = math.ceil(vx.rho * vx.k_in - 1e-9)
        in_total = 0.0
        for s, w in in_edges.get(v, []):
            in_total += w
        b0, b1 = layout.voxel_unit_base[v], layout.voxel_unit_base[v + 1]
        vn = sum(layout.units[u].neurons for u in range(b0, b1))
        if m > 0 and in_total > 0.0:
            for sv, w in in_edges.get(v, []):
                p_vox = w / in_total
                exc = float(layout.excitatory_count(sv))
                if exc <= 0.0:
                    continue
                picks_vox = float(vn) * m * p_vox
                for su in range(layout.voxel_unit_base[sv], layout.voxel_unit_base[sv + 1]):
                    if not layout.units[su].excitatory:
                        continue
                    n_u = float(layout.units[su].neurons)
                    picks_u = picks_vox * (n_u / exc)
                    bytes_ = rate_hz * dt_s * distinct(n_u, picks_u) * 4.0
                    for du in range(b0, b1):
                        share = float(layout.units[du].neurons) / float(vn)
                        traffic[su][du] += llround(bytes_ * share * 1e6)
        pmat = intra[vx.region]
        pops = len(vx.populations)
        for tp in range(pops):
            n_t = float(layout.units[b0 + tp].neurons)
            if n_t <= 0.0:
                continue
            wsum = 0.0
            for sp in range(pops):
                wsum += pmat[tp][sp] * float(layout.units[b0 + sp].neurons)
            if wsum <= 0.0:
                continue
            ppn = float(vx.k_in - m)
            for sp in range(pops):
                n_s = float(layout.units[b0 + sp].neurons)
                q = pmat[tp][sp] * n_s / wsum
                picks = n_t * ppn * q
                bytes_ = rate_hz * dt_s * distinct(n_s, picks) * 4.0
                traffic[b0 + sp][b0 + tp] += llround(bytes_ * 1e6)
    if byte_model == "b200_time":
        s1, s2, s3 = TIME_MODEL_FS[0], max(1, round(TIME_MODEL_FS[1] * rate_hz * dt_s)), 0
    else:
        s1, s2, s3 = BYTE_MODELS[byte_model]
    return UnitGraph(n, n * s1, n * kin * s2, n * s3, np.array(traffic, np.int64).reshape(U, U))


def _load(g: UnitGraph, cap: dict, u: int) -> float:
    return (cap["alpha"] * float(g.state_bytes[u]) + cap["beta"] * float(g.table_bytes[u]) +
            cap["mu"] * float(g.buffer_bytes[u]))


def validate_partition(unit_worker: List[int], workers: int, units: int):  # partition.cpp:27-42
    if workers == 0:
        raise ConfigError("partition with zero workers")
    if workers > 64:
        raise ConfigError("worker count exceeds the routing mask limit of 64")
    if len(unit_worker) != units:
        raise ConfigError("partition size does not match unit count")
    fill = [0] * workers
    for w in unit_worker:
        if w >= workers:
            raise ConfigError("partition worker id out of range")
        fill[w] += 1
    for w in range(workers):
        if fill[w] == 0:
            raise ConfigError(f"worker {w} has no units assigned")


def partition_sequential(g: UnitGraph, workers: int, cap: dict) -> List[int]:  # partition.cpp:311-344
    U = len(g.neurons)
    if workers == 0:
        raise ConfigError("zero workers")
    if U < workers:
        raise ConfigError("fewer units than workers")
    total = 0.0
    for u in range(U):
        total += _load(g, cap, u)
    share = cap["gamma"] if cap["gamma"] > 0.0 else total / workers
    out, w, cum = [0] * U, 0, 0.0
    for u in range(U):
        l = _load(g, cap, u)
        over = (cum + l > share) if cap["gamma"] > 0.0 else (cum + l > share * (w + 1) + 1e-9)
        left_after = U - u - 1
        if w + 1 < workers and over:
            w += 1
            if cap["gamma"] > 0.0:
                cum = 0.0
        if workers - 1 - w > left_after:
            raise ConfigError("sequential partition leaves a worker empty")
        out[u] = w
        cum += l
        if cap["gamma"] > 0.0 and cum > share:
            raise ConfigError(f"capacity budget cannot fit unit {u}")
    validate_partition(out, workers, U)
    return out


def partition_greedy(g: UnitGraph, workers: int, cap: dict) -> List[int]:  # partition.cpp:162-241
    U = len(g.neurons)
    if workers == 0:
        raise ConfigError("zero workers")
    if U < workers:
        raise ConfigError("fewer units than workers")
    loads = [_load(g, cap, u) for u in range(U)]
    order = sorted(range(U), key=lambda u: (-loads[u], u))
    T = g.traffic.copy()
    np.fill_diagonal(T, 0)  # i == u terms are skipped by the reference
    worker = np.full(U, -1, np.int64)
    recv = np.zeros(workers, np.int64)
    load = [0.0] * workers
    count = [0] * workers
    remaining = U
    # col[x] = sum of traffic[i][u] over placed i on x; row[x] = traffic[u][i]
    for u in order:
        empty = sum(1 for w in range(workers) if count[w] == 0)
        must_fill = empty >= remaining
        placed = worker >= 0
        col = np.zeros(workers, np.int64)
        row = np.zeros(workers, np.int64)
        if placed.any():
            np.add.at(col, worker[placed], T[placed, u])
            np.add.at(row, worker[placed], T[u, placed])
        col_sum = int(col.sum())
        best_w, best_f, best_load = -1, 0, 0.0
        for w in range(workers):
            if must_fill and count[w] != 0:
                continue
            new_load = load[w] + loads[u]
            if cap["gamma"] > 0.0 and new_load > cap["gamma"]:
                continue
            f = int(recv[w]) + col_sum - int(col[w])
            for x in range(workers):
                if x != w:
                    f = max(f, int(recv[x]) + int(row[x]))
            if best_w < 0 or f < best_f or (f == best_f and new_load < best_load):
                best_w, best_f, best_load = w, f, new_load
        if best_w < 0:
            raise ConfigError(f"capacity budget cannot fit unit {u}")
        w = best_w
        recv[w] += col_sum - int(col[w])
        for x in range(workers):
            if x != w:
                recv[x] += int(row[x])
        worker[u] = w
        load[w] += loads[u]
        count[w] += 1
        remaining -= 1
    out = worker.tolist()
    validate_partition(out, workers, U)
    return out


def partition_exact(g: UnitGraph, workers: int, cap: dict) -> List[int]:  # partition.cpp:243-309
    U = len(g.neurons)
    if workers == 0:
        raise ConfigError("zero workers")
    if U < workers:
        raise ConfigError("fewer units than workers")
    if U > 12:
        raise ConfigError("exact partitioning is limited to 12 units")
    ul = [_load(g, cap, u) for u in range(U)]
    T = g.traffic.tolist()
    assign, best, best_f = [0] * U, [], [2 ** 63 - 1]
    recv, load = [0] * workers, [0.0] * workers

    def dfs(u, used):
        if u == U:
            if used != workers:
                return
            f = max(recv)
            if f < best_f[0]:
                best_f[0] = f
                best[:] = assign
            return
        if workers - used > U - u:
            return
        for w in range(min(workers, used + 1)):
            new_load = load[w] + ul[u]
            if cap["gamma"] > 0.0 and new_load > cap["gamma"]:
                continue
            undo = [0] * workers
            for i in range(u):
                if assign[i] != w:
                    undo[w] += T[i][u]
                    undo[assign[i]] += T[u][i]
            partial = 0
            for x in range(workers):
                recv[x] += undo[x]
                partial = max(partial, recv[x])
            if partial < best_f[0]:
                assign[u] = w
                load[w] = new_load
                dfs(u + 1, max(used, w + 1))
                load[w] = new_load - ul[u]
            for x in range(workers):
                recv[x] -= undo[x]

    dfs(0, 0)
    if not best:
        raise ConfigError("no feasible partition under the capacity budget")
    validate_partition(best, workers, U)
    return list(best)


def partition_objective(g: UnitGraph, unit_worker: List[int], workers: int) -> int:
    uw = np.asarray(unit_worker)
    cross = uw[:, None] != uw[None, :]
    recv = np.zeros(workers, np.int64)
    np.add.at(recv, uw, (g.traffic * cross).sum(axis=0))
    return int(recv.max()) if workers else 0


def load_partition(path: str, units: int) -> tuple:  # partition.cpp:363-386
    with open(path) as f:
        t = f.read().split()
    try:
        if t[0] != "workers":
            raise ConfigError("partition file: expected 'workers N'")
        workers = int(t[1])
        if t[2] != "units" or int(t[3]) != units:
            raise ConfigError("partition file: unit count mismatch")
        out = []
        for i in range(units):
            if int(t[4 + 2 * i]) != i:
                raise ConfigError("partition file: bad unit line")
            out.append(int(t[5 + 2 * i]))
    except (IndexError, ValueError):
        raise ConfigError("partition file: bad unit line")
    validate_partition(out, workers, units)
    return out, workers


# ------------------------------------------------------------------ build
POP_DTYPE = np.dtype({
    "names": ["g_location", "g_scale", "weight_mean", "weight_spread", "split_ratio",
              "capacitance", "g_leak", "e_leak", "v_threshold", "v_reset",
              "refractory_steps", "e_rev", "tau", "omega", "ou_mean", "ou_sigma", "ou_tau",
              "excitatory", "dual_receptor"],
    "formats": [("<f8", 4), ("<f8", 4), ("<f8", 4), ("<f8", 4), "<f8", "<f4", "<f4", "<f4",
                "<f4", "<f4", "<u4", ("<f4", 4), ("<f4", 4), ("<f4", 4), "<f4", "<f4", "<f4",
                "u1", "u1"],
    "offsets": [0, 32, 64, 96, 128, 136, 140, 144, 148, 152, 156, 160, 176, 192, 208, 212, 216,
                220, 221],
    "itemsize": 224,
})
VOXEL_DTYPE = np.dtype({"names": ["k_in", "region", "rho", "unit_begin", "unit_end"],
                        "formats": ["<u4", "<u4", "<f8", "<u4", "<u4"],
                        "offsets": [0, 4, 8, 16, 20], "itemsize": 24})
EDGE_DTYPE = np.dtype({"names": ["src", "dst", "weight"], "formats": ["<u4", "<u4", "<f8"],
                       "offsets": [0, 4, 8], "itemsize": 16})


class NetSpecC(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_voxels", C.c_uint32), ("n_units", C.c_uint32),
                ("n_edges", C.c_uint32), ("n_workers", C.c_uint32), ("voxels", C.c_void_p),
                ("units", C.c_void_p), ("unit_pops", C.c_void_p), ("edges", C.c_void_p),
                ("intra", C.c_void_p * 4), ("intra_pops", C.c_uint32 * 4),
                ("unit_worker", C.c_void_p)]


@dataclass
class BuiltNetwork:
    """BuiltNetwork (pipeline.hpp:12-24) minus the sampled synapses, which
    live on the device."""
    cfg: dict
    graph: Connectome
    layout: Layout
    intra: dict
    unit_graph: Optional[UnitGraph]
    unit_worker: List[int]
    workers: int
    synapse_count: int
    arrays: dict

    def spec(self):
        a = self.arrays
        s = NetSpecC()
        s.seed = self.cfg["seed"]
        s.n_voxels, s.n_units = len(self.layout.voxels), len(self.layout.units)
        s.n_edges, s.n_workers = a["edges"].shape[0], self.workers
        s.voxels, s.units = ptr(a["voxels"]), ptr(a["units"])
        s.unit_pops, s.edges = ptr(a["pops"]), ptr(a["edges"])
        for r, name in enumerate(REGIONS):
            m = a["intra"][name]
            s.intra[r] = ptr(m) if m.size else None
            s.intra_pops[r] = m.shape[0] if m.size else 0
        s.unit_worker = ptr(a["unit_worker"])
        return s

    @property
    def total_neurons(self) -> int:
        return self.layout.total_neurons

    def unit_table(self) -> np.ndarray:
        return self.arrays["units"]


def build_network(cfg, workers: Optional[int] = None, method: Optional[str] = None) -> BuiltNetwork:
    """pipeline.cpp:98-125 up to (not including) sample_synapses/emit_tables."""
    cfg = parse_config(cfg)
    if workers is not None:
        cfg["workers"] = workers
    if method is not None:
        cfg["partition"]["method"] = method
    g = build_connectome(cfg)
    mc = None
    if "cortex" in g.region:
        path = cfg["microcolumn_path"] or os.environ.get("VOXSIM_MICROCOLUMN", "")
        if not path or not os.path.exists(path):
            raise ConfigError("network has cortex voxels but no micro-column file was found; "
                              "set microcolumn_path")
        mc = load_microcolumn(path)
    elif cfg["microcolumn_path"]:
        mc = load_microcolumn(cfg["microcolumn_path"])
    layout = build_layout(cfg, g, mc)
    intra = intra_matrices(mc)
    if len(g.edges) and g.voxel_count != len(layout.voxels):
        raise ConfigError("connectome / layout voxel count mismatch")
    p = cfg["partition"]
    W = cfg["workers"]
    ug = None
    if p["method"] == "even":
        uw = [u % W for u in range(len(layout.units))]
        validate_partition(uw, W, len(layout.units))
    elif p["method"] == "file":
        uw, W = load_partition(p["path"], len(layout.units))
    else:
        ug = build_unit_graph(layout, g, intra, p["rate_hz"], cfg["dt_ms"], p["byte_model"])
        if W == 1:
            uw = [0] * len(layout.units)
            validate_partition(uw, 1, len(layout.units))
        else:
            fn = {"greedy": partition_greedy, "sequential": partition_sequential,
                  "exact": partition_exact}[p["method"]]
            if p["byte_model"] in ("b200", "b200_time") and p["gamma"] <= 0:
                # per-GPU budget: the HBM budget, tightened to a near-even share
                # so the traffic objective cannot pile units onto one GPU
                total = sum(_load(ug, p, u) for u in range(len(layout.units)))
                cap = B200_HBM_BUDGET if p["byte_model"] == "b200" else float("inf")
                for slack in (1.1, 1.25, 1.5, 2.0, None):
                    q = dict(p)
                    q["gamma"] = cap if slack is None else min(cap, slack * total / W)
                    try:
                        uw = fn(ug, W, q)
                        break
                    except ConfigError:
                        if slack is None:
                            raise
            else:
                uw = fn(ug, W, p)
    # arrays for vxb_netspec
    units = np.zeros(len(layout.units), UNIT_DTYPE)
    pops = np.zeros(len(layout.units), POP_DTYPE)
    for i, u in enumerate(layout.units):
        units[i] = (u.gid_base, u.voxel, u.neurons, u.pop, int(u.excitatory), 0, 0)
        ps = layout.pop_of_unit(i)
        n = ps.neuron
        pops[i] = (ps.g_location, ps.g_scale, ps.weight_mean, ps.weight_spread, ps.split_ratio,
                   n.capacitance, n.g_leak, n.e_leak, n.v_threshold, n.v_reset,
                   n.refractory_steps, n.e_rev, n.tau, n.omega, ps.ou_mean, ps.ou_sigma,
                   ps.ou_tau, int(ps.excitatory), int(ps.dual_receptor))
    voxels = np.zeros(len(layout.voxels), VOXEL_DTYPE)
    for v, vx in enumerate(layout.voxels):
        voxels[v] = (vx.k_in, REGIONS.index(vx.region), vx.rho, layout.voxel_unit_base[v],
                     layout.voxel_unit_base[v + 1])
    edges = np.zeros(len(g.edges), EDGE_DTYPE)
    for i, e in enumerate(g.edges):
        edges[i] = e
    intra_arr = {r: np.ascontiguousarray(np.array(m, np.float64)) for r, m in intra.items()}
    syn = sum(u.neurons * layout.voxels[u.voxel].k_in for u in layout.units)
    if p["byte_model"] in ("b200", "b200_time"):  # every GPU must fit its share of the network
        s1, s2, s3 = BYTE_MODELS["b200"]
        load = [0.0] * W
        for u, x in enumerate(layout.units):
            load[uw[u]] += x.neurons * (s1 + s3 + layout.voxels[x.voxel].k_in * s2)
        budget = p["gamma"] if p["gamma"] > 0 and p["byte_model"] == "b200" else B200_HBM_BUDGET
        for w in range(W):
            if load[w] > budget:
                raise ConfigError(f"worker {w} needs {load[w] / 1e9:.1f} GB of HBM "
                                  f"(budget {budget / 1e9:.1f} GB)")
    arrays = {"units": units, "pops": pops, "voxels": voxels, "edges": edges,
              "intra": intra_arr, "unit_worker": np.asarray(uw, np.uint16)}
    return BuiltNetwork(cfg, g, layout, intra, ug, list(uw), W, syn, arrays)


B200_HBM_BYTES = 183e9   # one B200 (nvidia-smi: 183359 MiB... 179 GiB usable)
SORT_SLICE = 1 << 28      # entries per row-sort slice (Engine::sort_rows)


def memory_plan(net: "BuiltNetwork", record_raster: bool = False) -> list:
    """Per-rank device memory of the engine for `net` with one worker per
    rank (the allocations of csrc/vxb_engine.cu, l2_atomic path unless the
    shard fits the SM-tile path): resident bytes by buffer, the load-time
    scratch peak (generation counts, row-sort slices) and the total, against
    the 180 GB of a B200 (config 5 dry run)."""
    W = net.workers
    units = net.layout.units
    n_w = [0] * W
    syn_w = [0] * W
    for u, x in enumerate(units):
        n_w[net.unit_worker[u]] += x.neurons
        syn_w[net.unit_worker[u]] += x.neurons * net.layout.voxels[x.voxel].k_in
    N = sum(n_w)  # global sources: every rank indexes its out-CSR by global source
    out = []
    for r in range(W):
        n, S = n_w[r], syn_w[r]
        tile = W == 1 and n <= 148 * 6784 or W > 1 and n <= 148 * 6784
        res = {"neuron_state": 44 * n + (4 * n if tile else 0),  # V, j, I_ou(x2 tile), I_syn, g
               "pending": 32 * n, "dst_mask": 8 * n,
               "out_csr_offsets": 8 * (N + 1) + 4 * N,              # off + inner per global source
               "synapse_table": (8 if tile else 12) * S + 24,
               "spike_log": 4 * (min(n * 100, 1 << 29) if record_raster else 2 * n),
               "exchange_slots": 16 * (N - n) + 32 * W if W > 1 else 0}
        blocks = 1
        if not tile:
            n_ref = max(n_w)
            mb = 80 if (n_ref * 16 + (64 << 20) - 1) // (64 << 20) >= 6 else 64
            bn = (mb << 20) // 16
            blocks = 1 if n_ref <= bn else -(-n_ref // bn)
            if blocks > 1:
                res["l2_block_offsets"] = 4 * N * (blocks + 1)
        else:
            res["tile_segments"] = 16 * (S // 150 + N) + 2 * 8 * (S // 150)  # ~1 per 150 entries
        resident = sum(res.values())
        slice_ = min(S, SORT_SLICE)
        scratch = max(16 * (N + 1),                      # generation: counts + have-mask
                      12 * slice_ * 2 + 8 * (N + 1) if (blocks > 1 or tile) else 0)
        out.append({"rank": r, "neurons": n, "synapses": S, "path": "sm_tile" if tile else "l2_atomic",
                    "l2_blocks": blocks, "resident_bytes": resident, "load_scratch_bytes": scratch,
                    "peak_bytes": resident + scratch, "budget_bytes": B200_HBM_BYTES,
                    "fits": resident + scratch <= B200_HBM_BYTES, "buffers": res})
    return out


def hbm_bytes_per_worker(net: "BuiltNetwork") -> list:
    """Device bytes per worker under the B200 byte model."""
    s1, s2, s3 = BYTE_MODELS["b200"]
    load = [0] * net.workers
    for u, x in enumerate(net.layout.units):
        load[net.unit_worker[u]] += x.neurons * (s1 + s3 + net.layout.voxels[x.voxel].k_in * s2)
    return load


def sim_options_from(cfg: dict, **over) -> SimOptions:  # pipeline.cpp:127-137
    cfg = parse_config(cfg) if "connectome" not in cfg or isinstance(cfg, str) else cfg
    o = SimOptions(steps=cfg["steps"], dt_ms=cfg["dt_ms"], scheduler=cfg["scheduler"],
                   transport=cfg["transport"], workers_per_node=cfg["workers_per_node"],
                   recv_timeout_ms=cfg["recv_timeout_ms"], probe_gids=list(cfg["probe_gids"]))
    for k, v in over.items():
        setattr(o, k, v)
    return o


class GeneratedSimInstance(SimInstance):
    """SimInstance over a network sampled on the device (vxb_create_generated)."""

    def __init__(self, net: BuiltNetwork, options: SimOptions):
        self._lib = _abi.load_library()
        self._opt = options
        self._units = net.arrays["units"].copy()
        self._n_voxels = len(net.layout.voxels)
        self._hemo_every = 0
        self._net = net
        spec = net.spec()
        opt, keep = options._descriptor()
        h = C.c_void_p()
        rc = self._lib.vxb_create_generated(C.byref(spec), C.byref(opt), C.byref(h))
        del keep
        if rc != 0:
            from .engine import _raise
            _raise(rc, self._lib.vxb_last_error(None).decode())
        self._h = h

    def _member_args(self):
        spec = self._net.spec()
        return None, C.byref(spec), spec


def generate_tables(net: BuiltNetwork, device: int = 0) -> NetworkTables:
    """emit_tables output (WorkerTables with in-rows) for a small network,
    sampled on the device — for parity checks and file export."""
    lib = _abi.load_library()
    spec = net.spec()
    workers = []
    ulb = np.zeros(len(net.layout.units), np.uint32)
    fill = [0] * net.workers
    for u, x in enumerate(net.layout.units):
        w = net.unit_worker[u]
        ulb[u] = fill[w]
        fill[w] += x.neurons
    nsyn = [0] * net.workers
    for u, x in enumerate(net.layout.units):
        nsyn[net.unit_worker[u]] += x.neurons * net.layout.voxels[x.voxel].k_in
    for w in range(net.workers):
        neurons = np.zeros(fill[w], NEURON_DTYPE)
        syn = np.zeros(nsyn[w], SYN_DTYPE)
        rb = np.zeros(fill[w] + 1, np.uint64)
        rc = lib.vxb_generate_worker_table(C.byref(spec), device, w, ptr(neurons), fill[w],
                                           ptr(syn), nsyn[w], ptr(rb))
        if rc != 0:
            from .engine import _raise
            _raise(rc, lib.vxb_last_error(None).decode())
        workers.append(WorkerTable(w, net.workers, net.cfg["seed"], neurons, syn, rb))
    return NetworkTables(workers, net.arrays["unit_worker"].copy(), ulb, net.arrays["units"].copy(),
                         len(net.layout.voxels))


# ----------------------------------------------------------- one rank per GPU
def exchange_masks(local_bitmaps, rank: int, world: int, all_gather):
    """All-to-all of destination-mask bitmaps.

    local_bitmaps[h] = this rank's bitmap over shard h's neurons (bit i: neuron
    i of shard h has a target here).  Returns, for every h != rank, the bitmap
    rank h built over *this* rank's neurons.  `all_gather(obj) -> list` is the
    host collective (torch.distributed gloo in production, a stub in tests).
    """
    gathered = all_gather(local_bitmaps)
    return {h: gathered[h][rank] for h in range(world) if h != rank}


class DistributedSimInstance(SimInstance):
    """SimInstance for one rank of a one-process-per-GPU run: rank r holds
    worker r of the partition (netgen.build_network(cfg, workers=world)).
    Every method is collective over the ranks, like the reference's workers
    stepping in lockstep (engine.cpp:662-709)."""

    def __init__(self, net: BuiltNetwork, options: SimOptions, rank: int, world: int,
                 all_gather=None, barrier=None):
        if net.workers != world:
            raise ConfigError("distributed engines need one worker per rank")
        if all_gather is None or barrier is None:
            import torch.distributed as dist

            def all_gather(obj):
                out = [None] * world
                dist.all_gather_object(out, obj)
                return out
            barrier = dist.barrier
        self._lib = lib = _abi.load_library()
        self._opt = options
        self._units = net.arrays["units"].copy()
        self._n_voxels = len(net.layout.voxels)
        self._hemo_every = 0
        self._all_gather = all_gather
        self.rank, self.world = rank, world
        spec = net.spec()
        opt, keep = options._descriptor()
        h = C.c_void_p()
        rc = lib.vxb_create_generated_rank(C.byref(spec), C.byref(opt), rank, world, C.byref(h))
        del keep
        if rc != 0:
            from .engine import _raise
            _raise(rc, lib.vxb_last_error(None).decode())
        self._h = h
        if world > 1:
            bitmaps = []
            for d in range(world):
                nb = int(lib.vxb_mask_bytes(h, d))
                b = np.zeros(max(nb, 1), np.uint8)
                lib.vxb_mask_out(h, d, ptr(b), b.size)
                bitmaps.append(b[:nb].tobytes())
            for d, bits in exchange_masks(bitmaps, rank, world, all_gather).items():
                arr = np.frombuffer(bits, np.uint8).copy() if bits else np.zeros(1, np.uint8)
                rc = lib.vxb_mask_in(h, d, ptr(arr), arr.size)
                if rc:
                    self._err(rc)
            hd = (C.c_ubyte * 64)()
            if lib.vxb_ipc_handle(h, C.cast(hd, C.c_void_p), 64) != 0:
                raise SimError("cannot export the receive region (CUDA IPC)")
            handles = all_gather(bytes(hd))
            buf = np.frombuffer(b"".join(handles), np.uint8).copy()
            rc = lib.vxb_connect_peers(h, ptr(buf), 64)
            if rc:
                self._err(rc)
            barrier()

    def crossing_matrix(self) -> np.ndarray:
        """Collective: the full [src worker][dst worker] matrix, each rank
        contributing the column of its own targets."""
        return np.sum(np.stack(self._all_gather(super().crossing_matrix())), axis=0,
                      dtype=np.uint64)

    def advance(self, steps: int, fetch: bool = True):
        """Collective advance.  With the BOLD readout on, the ranks add their
        voxel counts (each holds its own units' spikes) and every rank runs
        the hemodynamics on the totals (vxb_hemo_feed_counts).  With timing
        rows, the ranks exchange the wire bytes of the batches they sent so
        every row carries its received bytes too (engine.cpp:495-523)."""
        if self.world > 1 and self._opt.record_timings:
            rc = self._lib.vxb_advance(self._h, steps)
            if rc != 0:
                self._err(rc)
            sent = np.zeros((steps, self.world), np.uint64)
            if sent.size:
                self._lib.vxb_result_wire_bytes(self._h, ptr(sent), sent.size)
            parts = self._all_gather(sent)
            recv = np.ascontiguousarray(np.stack([p[:, self.rank] for p in parts], axis=1),
                                        np.uint64)
            if recv.size:
                rc = self._lib.vxb_set_recv_wire_bytes(self._h, ptr(recv), steps)
                if rc != 0:
                    self._err(rc)
            if not self._hemo_every:
                return self.result() if fetch else None
            r = self.result()
        elif not (self._hemo_every and self.world > 1):
            return super().advance(steps, fetch)
        else:
            r = super().advance(steps, fetch=True)
        parts = self._all_gather(r.voxel_counts)
        tot = np.ascontiguousarray(np.sum(np.stack(parts), axis=0, dtype=np.uint64)
                                   .astype(np.uint32))
        rc = self._lib.vxb_hemo_feed_counts(self._h, ptr(tot), steps)
        if rc != 0:
            self._err(rc)
        r.voxel_counts, r.bold = tot, self._bold(steps)
        return r if fetch else None


# ------------------------------------------------- benchmark network shapes
def dti_like_connectome(voxels: int = 200, total_neurons: int = 20_000_000,
                        sparsity: float = 0.0072, weight_sigma: float = 0.5,
                        size_sigma: float = 0.5, seed: int = 3) -> Connectome:
    """BASELINE.json config 3: a synthetic DTI-like voxel graph — the
    reference's uniform generator (connectome.cpp:82-114: 7.2 per mille edge
    density, lognormal edge weights, ring fallback for isolated voxels) with
    lognormal voxel sizes normalised to `total_neurons` (largest remainder).
    The reference cannot express per-voxel sizes through its generators
    (SURVEY.md D6); the result is written as a connectome *file*
    (connectome.hpp:64-75), which both engines load."""
    g = make_uniform(voxels, 1, sparsity, weight_sigma, 0.0, seed)
    base = mix_key(seed, 8, 4)
    w = [math.exp(size_sigma * stream_normal(base, v)) for v in range(voxels)]
    tot = sum(w)
    exact = [x / tot * total_neurons for x in w]
    counts = [int(e) for e in exact]
    order = sorted(range(voxels), key=lambda v: -(exact[v] - counts[v]))
    for k in range(total_neurons - sum(counts)):
        counts[order[k % voxels]] += 1
    g.neuron_count = [max(1, c) for c in counts]
    g.validate()
    return g


def write_connectome_file(g: Connectome, path) -> str:
    p = str(path)
    with open(p, "w") as f:
        f.write(save_connectome_text(g))
    return p
