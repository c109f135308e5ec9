"""Trace reports of the BASELINE configs, restated from the reference's
analysis module (/root/reference/proj/src/analysis.cpp) on the host:

* ``time_to_residual`` (analysis.cpp:260-270) -- config 2's time to the
  planted ground state: the first sweep count at which the best feasible
  target energy so far is within ``rho_max`` per logical spin of ``e_gs``;
* ``residual_curve`` (analysis.cpp:38-96) -- config 3's residual energy
  rho_E(t) = (E(t) - E_gs) / n_logical averaged over runs, with the
  reference's bootstrap 95 % CI (same RNG stream: mt19937_64 seeded with
  derive_seed(seed, bootstrap, 0), rng.hpp:36-83);
* ``feasible_series`` (analysis.cpp:243-249), ``decode`` (constraints.cpp:149-162).

They consume the records the engine streams (api.Trace / TraceRecord);
infeasible records need the target state (``store_states``).  Pinned against
the reference's own analysis.cpp through oracle/_ref (tests/test_reports.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .api import ConfigError

_M64 = (1 << 64) - 1


def _mix64(z: int) -> int:  # rng.hpp:13-19
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def derive_seed(master: int, purpose: int, index: int) -> int:  # rng.hpp:36-40
    return _mix64(_mix64(master ^ _mix64(purpose)) ^ index)


PURPOSE_BOOTSTRAP = 7  # rng.hpp:30


class MT19937_64:
    """std::mt19937_64 (the C++ standard's parameters), the reference's RngStream engine."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _M64
        for i in range(1, 312):
            p = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (p ^ (p >> 62)) + i) & _M64
        self.i = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.i = 0

    def __call__(self) -> int:
        if self.i >= 312:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64

    def below(self, n: int) -> int:  # rng.hpp:58-65, rejection sampling
        limit = _M64 - _M64 % n
        while True:
            x = self()
            if x < limit:
                return x % n


def decode(copies: Sequence[Sequence[int]], state: np.ndarray) -> Tuple[np.ndarray, bool]:
    """Majority vote per chain, ties broken by the chain's first copy; feasible
    iff every chain agrees (constraints.cpp:149-162)."""
    logical = np.empty(len(copies), dtype=np.int8)
    feasible = True
    for u, chain in enumerate(copies):
        v = state[list(chain)].astype(np.int64)
        s = int(v.sum())
        logical[u] = (1 if s > 0 else -1) if s != 0 else int(v[0])
        if np.any(v[1:] != v[:-1]):
            feasible = False
    return logical, feasible


def logical_energy(logical_model, s: np.ndarray) -> float:
    """energy() of ising.cpp:70-77: -sum J s_i s_j - sum h s_i, in coupling order."""
    n, cpl, fields = logical_model
    e = 0.0
    for i, j, w in cpl:
        e -= w * int(s[i]) * int(s[j])
    for i in range(n):
        e -= fields[i] * int(s[i])
    return e


@dataclass
class EnergySample:
    t: int
    f: float
    feasible: bool


def feasible_series(records) -> List[EnergySample]:
    return [EnergySample(int(r.sweep_count), float(r.f), bool(r.feasible)) for r in records]


def time_to_residual(series: Sequence[EnergySample], e_gs: float, n_logical: int,
                     rho_max: float) -> Optional[int]:
    best = math.inf
    for s in series:
        if not s.feasible:
            continue
        best = min(best, s.f)
        if (best - e_gs) / n_logical <= rho_max:
            return s.t
    return None


@dataclass
class ResidualPoint:
    t: int
    rho_e: float
    ci95: float = 0.0


@dataclass
class ResidualCurve:
    n_logical: int
    points: List[ResidualPoint]
    trials: int
    instances: int
    degenerate_ci: bool


def _percentile(values: List[float], q: float) -> float:  # analysis.cpp:26-32
    v = sorted(values)
    pos = q * (len(v) - 1)
    lo = int(pos)
    hi = min(lo + 1, len(v) - 1)
    return v[lo] + (pos - lo) * (v[hi] - v[lo])


def residual_curve(runs, copies, logical_model, n_logical: int, strict: bool = False,
                   bootstrap_resamples: int = 200, seed: int = 1) -> ResidualCurve:
    """runs: sequence of (records, e_gs, instance_id) -- the reference's
    ResidualInput -- optionally extended to (records, e_gs, instance_id,
    copies, logical_model) when instances differ (config 3: 64 instances);
    records carry sweep_count, f, feasible and (for infeasible ones) state."""
    if not runs:
        raise ConfigError("residual: no runs given")
    n_rounds = len(runs[0][0])
    for run in runs:
        if len(run[0]) != n_rounds:
            raise ConfigError("residual: traces have mismatched lengths")
    rho = np.full((len(runs), n_rounds), np.nan)
    for r, run in enumerate(runs):
        recs, e_gs = run[0], run[1]
        cp, lm = (run[3], run[4]) if len(run) >= 5 else (copies, logical_model)
        for k, rec in enumerate(recs):
            if strict and not rec.feasible:
                continue
            cost = float(rec.f) if rec.feasible else \
                logical_energy(lm, decode(cp, np.asarray(rec.state))[0])
            rho[r, k] = (cost - e_gs) / n_logical
    degenerate = len(runs) < 2
    curve = ResidualCurve(n_logical, [], len(runs), len({run[2] for run in runs}), degenerate)
    rng = MT19937_64(derive_seed(seed, PURPOSE_BOOTSTRAP, 0))
    for k in range(n_rounds):
        values = [float(x) for x in rho[:, k] if not math.isnan(x)]
        pt = ResidualPoint(int(runs[0][0][k].sweep_count), math.nan)
        curve.points.append(pt)
        if not values:
            continue
        s = 0.0
        for v in values:
            s += v
        pt.rho_e = s / len(values)
        if degenerate or len(values) < 2:
            continue
        means = []
        for _ in range(bootstrap_resamples):
            acc = 0.0
            for _ in range(len(values)):
                acc += values[rng.below(len(values))]
            means.append(acc / len(values))
        if means:
            pt.ci95 = 0.5 * (_percentile(means, 0.975) - _percentile(means, 0.025))
    return curve
