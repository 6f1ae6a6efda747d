"""Holding-time parameterisations and the hazard / shedding functions.

Parameter objects and moment inversions follow the reference
(/root/reference/pkg/src/spreadsim/hazards.py:45-81, 161-193).  The
function evaluations (``erfcx_stable``, ``lognormal_hazard``,
``weibull_hazard``, ``erlang_hazard``, ``shedding``) run the same device
code the fused step uses (csrc/fs_device.cuh), so a value seen here is the
value the engine sees.  Weibull and Erlang holding times are north_star
extensions with no reference counterpart (parity unpinned).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .errors import InvalidMomentsError

__all__ = [
    "LogNormalParams",
    "WeibullParams",
    "ErlangParams",
    "Shedding",
    "erfcx_stable",
    "lognormal_hazard",
    "weibull_hazard",
    "erlang_hazard",
    "lognormal_pdf",
    "lognormal_from_mean_median",
    "weibull_from_mean_median",
    "shedding",
]


@dataclass(frozen=True)
class LogNormalParams:
    """ln T ~ N(mu, sigma^2) (hazards.py:45-66)."""

    mu: float
    sigma: float

    def __post_init__(self) -> None:
        if not self.sigma > 0.0:
            raise ValueError(f"sigma must be > 0, got {self.sigma}")

    @property
    def mean(self) -> float:
        return math.exp(self.mu + 0.5 * self.sigma**2)

    @property
    def median(self) -> float:
        return math.exp(self.mu)

    @property
    def mode(self) -> float:
        return math.exp(self.mu - self.sigma**2)


@dataclass(frozen=True)
class WeibullParams:
    """Weibull(shape k, scale lam): h(t) = (k/lam) (t/lam)^(k-1)."""

    k: float
    lam: float

    def __post_init__(self) -> None:
        if not (self.k > 0.0 and self.lam > 0.0):
            raise ValueError("weibull shape and scale must be > 0")

    @property
    def mean(self) -> float:
        return self.lam * math.gamma(1.0 + 1.0 / self.k)

    @property
    def median(self) -> float:
        return self.lam * math.log(2.0) ** (1.0 / self.k)


@dataclass(frozen=True)
class ErlangParams:
    """Erlang(shape k, rate r): sum of k exponentials of rate r."""

    k: int
    rate: float

    def __post_init__(self) -> None:
        if int(self.k) != self.k or self.k < 1 or not self.rate > 0.0:
            raise ValueError("erlang needs an integer shape >= 1 and rate > 0")

    @property
    def mean(self) -> float:
        return self.k / self.rate


def lognormal_from_mean_median(mean: float, median: float) -> LogNormalParams:
    """mu = ln median, sigma = sqrt(2 ln(mean/median)) (hazards.py:69-81)."""
    if not mean > median > 0.0:
        raise InvalidMomentsError(f"need mean > median > 0, got mean={mean}, median={median}")
    return LogNormalParams(mu=math.log(median), sigma=math.sqrt(2.0 * math.log(mean / median)))


def weibull_from_mean_median(mean: float, median: float) -> WeibullParams:
    """Shape k solving mean/median = Gamma(1+1/k) / ln2^(1/k) (bisection),
    then lam = median / ln2^(1/k)."""
    if not (mean > 0.0 and median > 0.0):
        raise InvalidMomentsError("need positive moments")
    target = mean / median

    def ratio(k: float) -> float:
        return math.gamma(1.0 + 1.0 / k) / math.log(2.0) ** (1.0 / k)

    lo, hi = 0.2, 50.0
    if not ratio(hi) < target < ratio(lo):
        raise InvalidMomentsError(f"mean/median={target} outside the Weibull range")
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if ratio(mid) > target:
            lo = mid
        else:
            hi = mid
    k = 0.5 * (lo + hi)
    return WeibullParams(k=k, lam=median / math.log(2.0) ** (1.0 / k))


@dataclass(frozen=True)
class Shedding:
    """Transmission profile s(tau) (hazards.py:161-193)."""

    kind: str
    params: LogNormalParams | None = None

    def __post_init__(self) -> None:
        if self.kind not in ("constant", "lognormal_hazard", "density_peak"):
            raise ValueError(f"unknown shedding kind {self.kind!r}")
        if self.kind != "constant" and self.params is None:
            raise ValueError(f"shedding kind {self.kind!r} requires params")

    @classmethod
    def constant(cls) -> "Shedding":
        return cls(kind="constant")

    @classmethod
    def lognormal_hazard(cls, params: LogNormalParams) -> "Shedding":
        return cls(kind="lognormal_hazard", params=params)

    @classmethod
    def density_peak(cls, params: LogNormalParams) -> "Shedding":
        return cls(kind="density_peak", params=params)


def lognormal_pdf(tau, p: LogNormalParams):
    """Log-normal density, 0 at tau = 0 (hazards.py:149-158); scalar host
    helper used for the density-peak normaliser."""
    t = np.atleast_1d(np.asarray(tau, dtype=np.float64))
    out = np.zeros_like(t)
    pos = t > 0.0
    if pos.any():
        tp = t[pos]
        zs = (np.log(tp) - p.mu) / p.sigma
        out[pos] = np.exp(-0.5 * zs * zs) / (tp * p.sigma * math.sqrt(2.0 * math.pi))
    return float(out[0]) if np.ndim(tau) == 0 else out


def _device_eval(x, fill) -> np.ndarray | float:
    arr = np.asarray(x, dtype=np.float64)
    scalar = arr.ndim == 0
    flat = np.ascontiguousarray(np.atleast_1d(arr).ravel())
    dev = _device.device()
    xin = torch.from_numpy(flat).to(dev)
    out = torch.empty_like(xin)
    fill(xin, out, _device.stream_handle(dev))
    res = out.cpu().numpy().reshape(np.atleast_1d(arr).shape)
    return float(res.ravel()[0]) if scalar else res


def erfcx_stable(z):
    """Piecewise scaled complementary error function (hazards.py:108-119)."""
    lib = _lib.load()
    return _device_eval(z, lambda a, b, s: _lib.check(lib.fs_erfcx_eval(a.data_ptr(), a.numel(), b.data_ptr(), s)))


def _hazard(tau, kind: int, p0: float, p1: float, precision: int = _lib.HAZ_F64):
    if np.any(np.atleast_1d(np.asarray(tau, dtype=np.float64)) < 0.0):
        raise ValueError("tau must be >= 0")
    lib = _lib.load()
    comp = _lib.FsCompartment(succ=0, terminal=0, hazard=kind, pad_=0, p0=p0, p1=p1)
    return _device_eval(
        tau, lambda a, b, s: _lib.check(lib.fs_hazard_eval(comp, a.data_ptr(), a.numel(), b.data_ptr(), precision, s))
    )


_HAZ_PRECISION = {"f64": _lib.HAZ_F64, "f32": _lib.HAZ_F32}


def lognormal_hazard(tau, p: LogNormalParams, precision: str = "f64"):
    """h(tau) = sqrt(2/pi) / (tau sigma erfcx(z)), h(0) = 0 (hazards.py:135-146).

    `precision` selects the engine's evaluation: "f64" is the reference's
    float64 arithmetic, "f32" the kernel's `hazard_precision="f32"` path
    (both returned as float64 arrays)."""
    return _hazard(tau, _lib.HZ_LOGNORMAL, p.mu, p.sigma, _HAZ_PRECISION[precision])


def weibull_hazard(tau, p: WeibullParams, precision: str = "f64"):
    return _hazard(tau, _lib.HZ_WEIBULL, p.k, p.lam, _HAZ_PRECISION[precision])


def erlang_hazard(tau, p: ErlangParams, precision: str = "f64"):
    return _hazard(tau, _lib.HZ_ERLANG, float(p.k), p.rate, _HAZ_PRECISION[precision])


def shedding(s: Shedding, tau):
    """s(tau) of a profile (hazards.py:196-218)."""
    t = np.asarray(tau, dtype=np.float64)
    if np.any(np.atleast_1d(t) < 0.0):
        raise ValueError("tau must be >= 0")
    if s.kind == "constant":
        return 1.0 if t.ndim == 0 else np.ones_like(t)
    if s.kind == "lognormal_hazard":
        return lognormal_hazard(tau, s.params)
    return lognormal_pdf(tau, s.params) / lognormal_pdf(s.params.mode, s.params)
