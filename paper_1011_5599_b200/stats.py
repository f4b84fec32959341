"""Statistics derived from N(t) (stats.hpp): host arithmetic on O(T) doubles.

``distribution_from_cdf`` and ``effective_diameter`` call the C++
implementations in libhanf.so (same code the C++ wrapper uses); the rest is
restated here in Python with the reference's evaluation order.
"""
from __future__ import annotations

import ctypes
import math
from ctypes import POINTER, c_double
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._lib import check, lib

K_RSD_CONSTANT = 1.06  # stats.hpp:120


@dataclass
class DistanceCdf:
    values: List[float] = field(default_factory=list)


@dataclass
class DistanceDistribution:
    density: List[float] = field(default_factory=list)
    mean: float = 0.0
    variance: float = 0.0
    spid: float = 0.0


def _arr(nf: Sequence[float]) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(nf, dtype=np.float64))


def cdf_from_nf(nf: Sequence[float]) -> DistanceCdf:
    """stats.hpp:33-42: H(t) = N(t)/N(T)."""
    if len(nf) == 0:
        raise ValueError("cdf: empty neighbourhood function")
    last = float(nf[-1])
    if not last > 0.0:
        raise ValueError("cdf: neighbourhood function is all zero")
    return DistanceCdf([float(v) / last for v in nf])


def distribution_from_cdf(cdf: DistanceCdf) -> DistanceDistribution:
    """stats.hpp:44-60: density, mean, variance, spid = variance/mean."""
    density, prev = [], 0.0
    for v in cdf.values:
        density.append(v - prev)
        prev = v
    # mean/variance/spid from the shared C++ implementation (nf == cdf works:
    # the cdf is its own normalisation)
    a = _arr(cdf.values)
    mean, var, spid = c_double(), c_double(), c_double()
    check(lib().hanf_distance_distribution(a.ctypes.data_as(POINTER(c_double)), a.size,
                                           ctypes.byref(mean), ctypes.byref(var),
                                           ctypes.byref(spid)))
    return DistanceDistribution(density, mean.value, var.value, spid.value)


def distance_distribution(nf: Sequence[float]) -> DistanceDistribution:
    """distribution_from_cdf(cdf_from_nf(nf)) in one call (bit-identical to
    the reference's two-step evaluation)."""
    a = _arr(nf)
    cdf = cdf_from_nf(a)
    density, prev = [], 0.0
    for v in cdf.values:
        density.append(v - prev)
        prev = v
    mean, var, spid = c_double(), c_double(), c_double()
    check(lib().hanf_distance_distribution(a.ctypes.data_as(POINTER(c_double)), a.size,
                                           ctypes.byref(mean), ctypes.byref(var),
                                           ctypes.byref(spid)))
    return DistanceDistribution(density, mean.value, var.value, spid.value)


def effective_diameter(nf: Sequence[float], alpha: float = 0.9,
                       interpolated: bool = False) -> float:
    """stats.hpp:65-77."""
    a = _arr(nf)
    out = c_double()
    check(lib().hanf_effective_diameter(a.ctypes.data_as(POINTER(c_double)), a.size,
                                        float(alpha), int(bool(interpolated)),
                                        ctypes.byref(out)))
    return out.value


@dataclass
class DiameterInterval:
    lo: Optional[int] = None
    hi: Optional[int] = None
    confidence: float = 1.0
    note: str = ""


def diameter_interval(nf: Sequence[float], alpha: float, epsilon: float,
                      delta: float) -> DiameterInterval:
    """stats.hpp:88-116 (Algorithm 3 interval form)."""
    if not (0.0 < alpha <= 1.0):
        raise ValueError("diameter interval: alpha must be in (0, 1]")
    if epsilon < 0.0 or delta < 0.0 or delta >= 1.0:
        raise ValueError("diameter interval: bad epsilon/delta")
    if len(nf) == 0:
        raise ValueError("diameter interval: empty input")
    out = DiameterInterval(confidence=1.0 - 3.0 * delta)
    mx = float(nf[-1])
    lo_t = alpha * (1.0 - 2.0 * epsilon)
    hi_t = alpha * (1.0 + 2.0 * epsilon)
    for t, v in enumerate(nf):
        if float(v) / mx <= lo_t:
            out.lo = t
    if hi_t > 1.0:
        out.note = ("upper bound undefined: alpha(1+2eps) exceeds 1, no point of the cdf "
                    "can reach it")
        return out
    for t, v in enumerate(nf):
        if float(v) / mx >= hi_t:
            out.hi = t
            break
    return out


@dataclass
class PrecisionSpec:
    """stats.hpp:122-145."""
    m: int = 0
    eta: float = 0.0
    epsilon: Optional[float] = None
    delta: Optional[float] = None

    def chebyshev_confidence(self, eps: float) -> float:
        return max(0.0, 1.0 - self.eta * self.eta / (eps * eps))

    def vp_confidence(self, eps: float) -> float:
        return max(0.0, 1.0 - 4.0 * self.eta * self.eta / (9.0 * eps * eps))

    def ksigma_error(self, k: float) -> float:
        return k * self.eta

    @staticmethod
    def ksigma_confidence(k: float) -> float:
        return 1.0 - 4.0 / (9.0 * k * k)

    def memory_bits(self, n: int) -> float:
        reg_bits = math.ceil(math.log2(math.log2(float(n))))
        return float(self.m) * reg_bits * float(n)

    def memory_gib(self, n: int) -> float:
        return self.memory_bits(n) / 8.0 / (1024.0 * 1024.0 * 1024.0)


def precision_from_m(m: int) -> PrecisionSpec:
    """stats.hpp:155-162."""
    if m < 16 or (m & (m - 1)) != 0:
        raise ValueError("precision: m must be a power of two >= 16")
    return PrecisionSpec(m=m, eta=K_RSD_CONSTANT / math.sqrt(float(m)))


def precision_from_eta(eta: float) -> PrecisionSpec:
    """stats.hpp:164-170."""
    if not (0.0 < eta < 1.0):
        raise ValueError("precision: eta must be in (0, 1)")
    target = 1.12 / (eta * eta)
    m = 16
    while float(m) < target:
        m <<= 1
    return precision_from_m(m)


def precision_from_error(epsilon: float, delta: float) -> PrecisionSpec:
    """stats.hpp:174-183."""
    if not (0.0 < epsilon < 1.0) or not (0.0 < delta < 1.0):
        raise ValueError("precision: epsilon and delta must be in (0, 1)")
    eta = epsilon * math.sqrt(delta)
    if eta >= 1.0:
        raise ValueError("precision: infeasible inputs")
    spec = precision_from_eta(eta)
    spec.epsilon, spec.delta = epsilon, delta
    return spec


@dataclass
class RunSummary:
    seed: int = 0
    avg_distance: float = 0.0
    spid: float = 0.0
    ied: float = 0.0


@dataclass
class MultiRunReport:
    n: int = 0
    m: int = 0
    alpha: float = 0.9
    per_run: List[RunSummary] = field(default_factory=list)
    mean: RunSummary = field(default_factory=RunSummary)
    stddev: RunSummary = field(default_factory=RunSummary)
    mean_nf: List[float] = field(default_factory=list)


def aggregate_runs(runs, alpha: float = 0.9) -> MultiRunReport:
    """stats.hpp:205-257: per-run ad/spid/ied with mean and sample sd."""
    if len(runs) < 2:
        raise ValueError("aggregate: need at least two runs")
    for run in runs:
        if run.n != runs[0].n or run.m != runs[0].m:
            raise ValueError("aggregate: runs disagree on graph or m")
    rep = MultiRunReport(n=runs[0].n, m=runs[0].m, alpha=alpha)
    longest = max(len(r.values) for r in runs)
    rep.mean_nf = [0.0] * longest
    for run in runs:
        dist = distance_distribution(run.values)
        rep.per_run.append(RunSummary(run.seed, dist.mean, dist.spid,
                                      effective_diameter(run.values, alpha, True)))
        for t in range(longest):
            rep.mean_nf[t] += run.values[t] if t < len(run.values) else run.values[-1]
    r = float(len(runs))
    rep.mean_nf = [v / r for v in rep.mean_nf]

    def moments(get):
        mean = 0.0
        for s in rep.per_run:
            mean += get(s)
        mean /= r
        ss = 0.0
        for s in rep.per_run:
            d = get(s) - mean
            ss += d * d
        return mean, math.sqrt(ss / (r - 1.0))

    rep.mean.avg_distance, rep.stddev.avg_distance = moments(lambda s: s.avg_distance)
    rep.mean.spid, rep.stddev.spid = moments(lambda s: s.spid)
    rep.mean.ied, rep.stddev.ied = moments(lambda s: s.ied)
    return rep
