"""Data assimilation over the B200 engine: the reference's ensemble loop
(/root/reference/proj/src/assim.cpp, assim.hpp) driving device members.

The loop itself is host arithmetic on a few dozen numbers per window and
stays a restatement of the reference; what changes is what it drives:

* every ``EnsembleMember`` is a member engine that views the donor's synapse
  tables on the GPU (``SimInstance.member``, vxb_create_member) instead of
  holding its own copy, so an ensemble of config-2 members costs one 12 GB
  table;
* each window's BOLD sample comes from the device readout
  (``set_hemodynamics`` with ``sample_every = window_steps``: the reference's
  ``window_bold``, assim.cpp:51-71), not from rates copied to the host.

Conductances are drawn on the host exactly as the reference draws them
(``netgen.sample_conductances_exact``, glibc ``log``/``cos``/``exp``), so a
member's spikes are the reference member's spikes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import netgen
from .engine import ConfigError, HemoParams, SimInstance

RNG_ASSIM = 9  # rngstream::assim (rng.hpp:27)


@dataclass
class AssimTarget:
    """AssimTarget (assim.hpp:15-19): a (unit, receptor) log-space location."""
    unit: int = 0
    receptor: int = 0


@dataclass
class AssimOptions:
    """AssimOptions (assim.hpp:21-37)."""
    members: int = 8
    windows: int = 50
    window_steps: int = 800
    dt_ms: float = 1.0
    obs_noise_sd: float = 2e-4
    inflation: float = 1.05
    min_spread: float = 1e-3
    prior_sd: float = 0.25
    baseline_hz: float = 5.0
    divergence_patience: int = 5
    divergence_factor: float = 10.0
    seed: int = 1
    hemo: HemoParams = field(default_factory=HemoParams)
    targets: List[AssimTarget] = field(default_factory=list)


@dataclass
class AssimWindowStat:
    """AssimWindowStat (assim.hpp:39-45)."""
    window: int
    innovation_rms: float
    pearson_r: float
    mean_spread: float
    target_mean: List[float]


@dataclass
class AssimResult:
    """AssimResult (assim.hpp:47-53)."""
    windows: List[AssimWindowStat]
    final_mean: List[float]
    final_spread: List[float]
    diverged: bool = False
    diverged_window: int = 0


def validate_assim(o: AssimOptions) -> None:
    """validate_assim (assim.cpp:40-49)."""
    if o.members < 2:
        raise ConfigError("assimilation needs >= 2 members")
    if o.window_steps == 0:
        raise ConfigError("window_steps must be >= 1")
    if not o.targets:
        raise ConfigError("no assimilation targets")
    if not o.obs_noise_sd > 0:
        raise ConfigError("obs_noise_sd must be > 0")
    if o.inflation < 1.0:
        raise ConfigError("inflation must be >= 1")
    if not o.baseline_hz > 0:
        raise ConfigError("baseline_hz must be > 0")


def pearson(a: Sequence[float], b: Sequence[float]) -> float:
    """assim.cpp:21-40, summation order kept."""
    n = len(a)
    if n < 2:
        return 0.0
    ma = mb = 0.0
    for x, y in zip(a, b):
        ma += x
        mb += y
    ma /= n
    mb /= n
    saa = sbb = sab = 0.0
    for x, y in zip(a, b):
        saa += (x - ma) * (x - ma)
        sbb += (y - mb) * (y - mb)
        sab += (x - ma) * (y - mb)
    if saa <= 0 or sbb <= 0:
        return 0.0
    return sab / math.sqrt(saa * sbb)


def ensrf_update(ensemble: List[List[float]], forecasts: List[List[float]],
                 obs: Sequence[float], obs_var: float, inflation: float,
                 min_spread: float) -> None:
    """EnsrfUpdate::apply (assim.cpp:108-179): serial deterministic
    square-root filter on the augmented state, in the reference's loop and
    summation order (scalar doubles, so results match it bit for bit)."""
    m = len(ensemble)
    if m < 2 or len(forecasts) != m:
        raise ConfigError("ensemble and forecasts must have >= 2 members")
    p, q = len(ensemble[0]), len(obs)
    z = []
    for i in range(m):
        if len(forecasts[i]) != q:
            raise ConfigError("forecast size does not match observations")
        z.append(list(ensemble[i]) + [float(x) for x in forecasts[i]])
    mean = [0.0] * (p + q)
    dev_y = [0.0] * m
    for o in range(q):
        yc = p + o
        for c in range(p + q):
            acc = 0.0
            for i in range(m):
                acc += z[i][c]
            mean[c] = acc / m
        s_yy = 0.0
        for i in range(m):
            dev_y[i] = z[i][yc] - mean[yc]
            s_yy += dev_y[i] * dev_y[i]
        s_yy /= (m - 1)
        denom = s_yy + obs_var
        if denom <= 0:
            continue
        innov = obs[o] - mean[yc]
        alpha = 1.0 / (1.0 + math.sqrt(obs_var / denom))
        for c in range(p + q):
            cov = 0.0
            for i in range(m):
                cov += (z[i][c] - mean[c]) * dev_y[i]
            cov /= (m - 1)
            gain = cov / denom
            new_mean = mean[c] + gain * innov
            for i in range(m):
                dev = (z[i][c] - mean[c]) - alpha * gain * dev_y[i]
                z[i][c] = new_mean + dev
    for c in range(p):
        mu = 0.0
        for i in range(m):
            mu += z[i][c]
        mu /= m
        var = 0.0
        for i in range(m):
            var += (z[i][c] - mu) * (z[i][c] - mu)
        sd = math.sqrt(var / (m - 1))
        scale = inflation
        if sd * inflation < min_spread:
            scale = min_spread / sd if sd > 0 else 0.0
        for i in range(m):
            dev = (z[i][c] - mu) * scale
            if sd == 0.0 and min_spread > 0:
                centered = (i - 0.5 * (m - 1)) / max(1.0, 0.5 * (m - 1))
                dev = min_spread * centered
            ensemble[i][c] = mu + dev


class EnsembleMember:
    """EnsembleMember (assim.hpp:55-76, assim.cpp:74-107) on a member engine
    that shares `donor`'s synapse tables; BOLD from the device readout."""

    def __init__(self, donor: SimInstance, units: np.ndarray, opts: AssimOptions,
                 member_index: int, scales: Sequence[float]):
        self.sim = donor.member()
        self.sim.set_hemodynamics(opts.hemo, opts.baseline_hz, opts.window_steps)
        self.units, self.opts, self.member = units, opts, member_index
        for t in opts.targets:
            if t.unit >= len(units):
                raise ConfigError("assimilation target unit out of range")
            if t.receptor < 0 or t.receptor >= 4:
                raise ConfigError("assimilation target receptor out of range")
        self.scales = list(scales)

    def run_window(self, params: Sequence[float], window: int) -> np.ndarray:
        o = self.opts
        if len(params) != len(o.targets):
            raise ConfigError("parameter vector size does not match targets")
        salt = netgen.mix_key((self.member + 1) & (2**64 - 1), window + 1)
        for i, t in enumerate(o.targets):
            count = int(self.units[t.unit]["neurons"])
            self.sim.set_conductances(t.unit, t.receptor, netgen.sample_conductances_exact(
                o.seed, salt, t.unit, t.receptor, params[i], self.scales[i], count))
        r = self.sim.advance(o.window_steps)
        return r.bold[-1]

    def close(self):
        self.sim.close()


def _prior(opts: AssimOptions, locations: Sequence[float]) -> List[List[float]]:
    """Initial ensemble around the generation-time prior (assim.cpp:204-214)."""
    params = [[0.0] * len(opts.targets) for _ in range(opts.members)]
    for k, t in enumerate(opts.targets):
        base = netgen.mix_key(netgen.mix_key(opts.seed, RNG_ASSIM, t.unit), t.receptor)
        for i in range(opts.members):
            params[i][k] = locations[k] + opts.prior_sd * netgen.stream_normal(base, i)
    return params


def assimilate(donor: SimInstance, units: np.ndarray, observed: np.ndarray,
               opts: AssimOptions, locations: Sequence[float],
               scales: Sequence[float]) -> AssimResult:
    """assimilate (assim.cpp:181-299) with device members.  `donor` is an
    instance of the surrogate network (its tables are shared, its own state
    is not advanced); `locations` / `scales` are the targets' population
    g_location / g_scale (layout.pop_of_unit(unit), assim.cpp:86-89, 207)."""
    validate_assim(opts)
    opts.hemo  # validated by set_hemodynamics
    observed = np.asarray(observed, np.float64)
    windows = min(opts.windows, observed.shape[0])
    if windows == 0:
        raise ConfigError("no observation windows")
    voxels = donor._n_voxels
    if observed.shape[1] != voxels:
        raise ConfigError("observed BOLD row does not match voxel count")
    members = [EnsembleMember(donor, units, opts, i, scales) for i in range(opts.members)]
    try:
        params = _prior(opts, locations)
        p = len(opts.targets)
        res = AssimResult([], [0.0] * p, [0.0] * p)
        first_rms, bad = -1.0, 0
        obs_var = opts.obs_noise_sd * opts.obs_noise_sd
        for w in range(windows):
            forecasts = [list(map(float, members[i].run_window(params[i], w)))
                         for i in range(opts.members)]
            fmean = [0.0] * voxels
            for i in range(opts.members):
                for v in range(voxels):
                    fmean[v] += forecasts[i][v]
            for v in range(voxels):
                fmean[v] /= opts.members
            obs = [float(x) for x in observed[w]]
            rms = 0.0
            for v in range(voxels):
                d = obs[v] - fmean[v]
                rms += d * d
            innovation = math.sqrt(rms / voxels)
            r = pearson(fmean, obs)
            ensrf_update(params, forecasts, obs, obs_var, opts.inflation, opts.min_spread)
            tmean, spread = [], 0.0
            for k in range(p):
                mu = 0.0
                for i in range(opts.members):
                    mu += params[i][k]
                mu /= opts.members
                tmean.append(mu)
                var = 0.0
                for i in range(opts.members):
                    var += (params[i][k] - mu) * (params[i][k] - mu)
                spread += math.sqrt(var / (opts.members - 1))
            res.windows.append(AssimWindowStat(w, innovation, r, spread / p, tmean))
            if first_rms < 0:
                first_rms = max(res.windows[0].innovation_rms, 1e-12)
            bad = bad + 1 if innovation > opts.divergence_factor * first_rms else 0
            if opts.divergence_patience > 0 and bad >= opts.divergence_patience:
                res.diverged, res.diverged_window = True, w
                break
        for k in range(p):
            mu = 0.0
            for i in range(opts.members):
                mu += params[i][k]
            mu /= opts.members
            var = 0.0
            for i in range(opts.members):
                var += (params[i][k] - mu) * (params[i][k] - mu)
            res.final_mean[k], res.final_spread[k] = mu, math.sqrt(var / (opts.members - 1))
        return res
    finally:
        for m in members:
            m.close()


def run_forward_bold(donor: SimInstance, units: np.ndarray, opts: AssimOptions, windows: int,
                     true_params: Optional[Sequence[float]] = None,
                     scales: Sequence[float] = ()) -> np.ndarray:
    """run_forward_bold (assim.cpp:301-326) on a member engine: the truth of a
    twin experiment (member index -1) when `true_params` is given, else the
    table conductances; BOLD per (window, voxel)."""
    if true_params is not None:
        truth = EnsembleMember(donor, units, opts, -1, scales)
        try:
            return np.stack([truth.run_window(true_params, w) for w in range(windows)])
        finally:
            truth.close()
    sim = donor.member()
    try:
        sim.set_hemodynamics(opts.hemo, opts.baseline_hz, opts.window_steps)
        return np.stack([sim.advance(opts.window_steps).bold[-1] for _ in range(windows)])
    finally:
        sim.close()
