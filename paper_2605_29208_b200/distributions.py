"""Emission families on the hot path, as immutable parameter records.

Mirrors the value objects of the reference (distributions.py:164-537): the
same class names, field names, ``family`` tags, ``params()`` keys and
constructor validation messages, so models built against the reference API
carry over unchanged.  What changes is where the numbers are evaluated: a
distribution here is a record that the device kernels consume through
``record()`` -- the family id, the raw parameters and the per-state constants
the host computes with the reference's own scalar math (``math.log``,
``math.lgamma``, ``special.log_bessel_i0``), so IEEE-basic-op families
(Gaussian, Poisson) reproduce the reference bit for bit on the GPU.

The ten families off the benchmarked configurations (LogNormal, Exponential,
Rayleigh, Uniform, Categorical, Beta, Weibull, NegativeBinomial, ChiSquared,
Pareto; distributions.py:208-341, 393-511) are records
of the same kind: the device evaluates them in the runtime-family paths of
every kernel and fits them with the weighted-sample passes of
csrc/hmm_extfit.cuh.  Categorical keeps at most 8 categories on the device
(its log-probabilities fill the 8 parameter slots of the record).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import ClassVar

import numpy as np

from . import _native
from .special import log_bessel_i0, log_gamma

__all__ = [
    "Distribution",
    "Gaussian",
    "StudentT",
    "Gamma",
    "VonMises",
    "Poisson",
    "LogNormal",
    "Exponential",
    "Rayleigh",
    "Uniform",
    "Categorical",
    "Beta",
    "Weibull",
    "NegativeBinomial",
    "ChiSquared",
    "Pareto",
    "Joint",
    "EcmeConfig",
    "FitWarning",
    "FAMILIES",
    "SCALE_FLOOR",
    "VONMISES_KAPPA_CEILING",
]

LOG_2PI = math.log(2.0 * math.pi)
SCALE_FLOOR = 1e-9  # distributions.py:73
VONMISES_KAPPA_CEILING = 1e5  # distributions.py:74
NEGBINOM_R_CEILING = 1e6  # distributions.py:76
CATEGORICAL_MAX = 8  # categories a device record holds


class FitWarning(RuntimeWarning):
    """Raised as a warning when a fit hits an iteration cap or a boundary."""


@dataclass(frozen=True)
class EcmeConfig:
    """Controls for the Student-t conditional maximization steps (distributions.py:144-150)."""

    nu_ceiling: float = 1e6
    nu_tol: float = 1e-6
    max_newton: int = 50


def _check_finite(name: str, value: float) -> None:
    if not math.isfinite(value):
        raise ValueError(f"{name} must be finite, got {value}")


def _check_positive(name: str, value: float) -> None:
    _check_finite(name, value)
    if value <= 0.0:
        raise ValueError(f"{name} must be > 0, got {value}")


class Distribution:
    """Base of the emission records (distributions.py:164-184)."""

    family: ClassVar[str]
    param_count: ClassVar[int]

    def params(self) -> dict[str, float]:
        raise NotImplementedError

    def num_free_params(self) -> int:
        return self.param_count

    def record(self) -> tuple[int, list[float], list[float]]:
        """(family id, p[4], c[4]) for loghmm_emission_t."""
        raise NotImplementedError

    @property
    def n_streams(self) -> int:
        return 1

    def log_prob(self, y, dtype="float64"):
        """Natural-log density at y, evaluated by the device emission kernel
        (loghmm_emission); -inf outside the support."""
        from .inference import _single_state_log_prob

        return _single_state_log_prob(self, y, dtype)


@dataclass(frozen=True)
class Gaussian(Distribution):
    mu: float
    sigma: float

    family: ClassVar[str] = "gaussian"
    param_count: ClassVar[int] = 2

    def __post_init__(self):
        _check_finite("gaussian.mu", self.mu)
        _check_positive("gaussian.sigma", self.sigma)

    def params(self):
        return {"mu": self.mu, "sigma": self.sigma}

    def record(self):
        # distributions.py:199-201: (-0.5 * LOG_2PI - log(sigma)) is one Python float
        c0 = -0.5 * LOG_2PI - math.log(self.sigma)
        return _native.FAM["gaussian"], [self.mu, self.sigma, 0.0, 0.0], [c0, 0.0, 0.0, 0.0]


@dataclass(frozen=True)
class StudentT(Distribution):
    mu: float
    sigma: float
    nu: float

    family: ClassVar[str] = "student_t"
    param_count: ClassVar[int] = 3

    def __post_init__(self):
        _check_finite("student_t.mu", self.mu)
        _check_positive("student_t.sigma", self.sigma)
        _check_positive("student_t.nu", self.nu)

    def params(self):
        return {"mu": self.mu, "sigma": self.sigma, "nu": self.nu}

    def record(self):
        # distributions.py:526-534, scalar prefix evaluated left to right
        nu = self.nu
        c0 = (
            log_gamma((nu + 1.0) / 2.0)
            - log_gamma(nu / 2.0)
            - 0.5 * math.log(nu * math.pi)
            - math.log(self.sigma)
        )
        c1 = (nu + 1.0) / 2.0
        return _native.FAM["student_t"], [self.mu, self.sigma, nu, 0.0], [c0, c1, 0.0, 0.0]


@dataclass(frozen=True)
class Gamma(Distribution):
    shape: float
    rate: float

    family: ClassVar[str] = "gamma"
    param_count: ClassVar[int] = 2

    def __post_init__(self):
        _check_positive("gamma.alpha", self.shape)
        _check_positive("gamma.beta", self.rate)

    def params(self):
        return {"alpha": self.shape, "beta": self.rate}

    def record(self):
        # distributions.py:378-386
        c0 = self.shape * math.log(self.rate) - log_gamma(self.shape)
        c1 = self.shape - 1.0
        return _native.FAM["gamma"], [self.shape, self.rate, 0.0, 0.0], [c0, c1, 0.0, 0.0]


@dataclass(frozen=True)
class VonMises(Distribution):
    mu: float
    kappa: float

    family: ClassVar[str] = "von_mises"
    param_count: ClassVar[int] = 2

    def __post_init__(self):
        _check_finite("von_mises.mu", self.mu)
        _check_finite("von_mises.kappa", self.kappa)
        if self.kappa < 0:
            raise ValueError(f"von_mises.kappa must be >= 0, got {self.kappa}")
        if not (-math.pi < self.mu <= math.pi):
            raise ValueError(f"von_mises.mu must lie in (-pi, pi], got {self.mu}")

    def params(self):
        return {"mu": self.mu, "kappa": self.kappa}

    def record(self):
        # distributions.py:359-360
        return (
            _native.FAM["von_mises"],
            [self.mu, self.kappa, 0.0, 0.0],
            [LOG_2PI, log_bessel_i0(self.kappa), 0.0, 0.0],
        )


@dataclass(frozen=True)
class Poisson(Distribution):
    rate: float

    family: ClassVar[str] = "poisson"
    param_count: ClassVar[int] = 1

    def __post_init__(self):
        _check_positive("poisson.lambda", self.rate)

    def params(self):
        return {"lambda": self.rate}

    def record(self):
        # distributions.py:256-260
        return _native.FAM["poisson"], [self.rate, 0.0, 0.0, 0.0], [math.log(self.rate), 0.0, 0.0, 0.0]


def _rec(name, p, c, aux=0):
    p = list(p) + [0.0] * (4 - len(p))
    c = list(c) + [0.0] * (4 - len(c))
    return _native.FAM[name], p, c, aux


@dataclass(frozen=True)
class LogNormal(Distribution):
    mu: float
    sigma: float

    family: ClassVar[str] = "lognormal"
    param_count: ClassVar[int] = 2

    def __post_init__(self):
        _check_finite("lognormal.mu", self.mu)
        _check_positive("lognormal.sigma", self.sigma)

    def params(self):
        return {"mu": self.mu, "sigma": self.sigma}

    def record(self):
        # distributions.py:219-223: -ly - log(sigma) - 0.5*LOG_2PI - 0.5*z*z
        return _rec("lognormal", [self.mu, self.sigma], [math.log(self.sigma), 0.5 * LOG_2PI])


@dataclass(frozen=True)
class Exponential(Distribution):
    rate: float

    family: ClassVar[str] = "exponential"
    param_count: ClassVar[int] = 1

    def __post_init__(self):
        _check_positive("exponential.lambda", self.rate)

    def params(self):
        return {"lambda": self.rate}

    def record(self):
        # distributions.py:239-240: log(rate) - rate*y
        return _rec("exponential", [self.rate], [math.log(self.rate)])


@dataclass(frozen=True)
class Rayleigh(Distribution):
    sigma: float

    family: ClassVar[str] = "rayleigh"
    param_count: ClassVar[int] = 1

    def __post_init__(self):
        _check_positive("rayleigh.sigma", self.sigma)

    def params(self):
        return {"sigma": self.sigma}

    def record(self):
        # distributions.py:276-279: log(y) - log(s2) - y*y/(2*s2)
        s2 = self.sigma * self.sigma
        return _rec("rayleigh", [self.sigma], [math.log(s2), 2.0 * s2])


@dataclass(frozen=True)
class Uniform(Distribution):
    lower: float
    upper: float

    family: ClassVar[str] = "uniform"
    param_count: ClassVar[int] = 2

    def __post_init__(self):
        _check_finite("uniform.a", self.lower)
        _check_finite("uniform.b", self.upper)
        if not self.lower < self.upper:
            raise ValueError(f"uniform requires a < b, got a={self.lower}, b={self.upper}")

    def params(self):
        return {"a": self.lower, "b": self.upper}

    def record(self):
        # distributions.py:299-301
        return _rec("uniform", [self.lower, self.upper], [-math.log(self.upper - self.lower)])


@dataclass(frozen=True)
class Categorical(Distribution):
    probs: tuple

    family: ClassVar[str] = "categorical"
    param_count: ClassVar[int] = 0  # overridden per instance

    def __post_init__(self):
        probs = tuple(float(p) for p in self.probs)
        if len(probs) < 1:
            raise ValueError("categorical requires at least one category")
        for k, p in enumerate(probs):
            _check_finite(f"categorical.p{k}", p)
            if p < 0:
                raise ValueError(f"categorical.p{k} must be >= 0, got {p}")
        if abs(sum(probs) - 1.0) > 1e-12:
            raise ValueError(f"categorical probabilities must sum to 1 within 1e-12, got {sum(probs)}")
        object.__setattr__(self, "probs", probs)

    def params(self):
        return {f"p{k}": p for k, p in enumerate(self.probs)}

    def num_free_params(self) -> int:
        return len(self.probs) - 1

    def record(self):
        # distributions.py:328-334: log p_k (np.log, -inf for p_k = 0) in the 8 slots
        m = len(self.probs)
        if m > CATEGORICAL_MAX:
            raise ValueError(f"categorical with {m} categories: the device record holds at most "
                             f"{CATEGORICAL_MAX}")
        with np.errstate(divide="ignore"):
            lp = [float(np.log(p)) if p > 0 else -math.inf for p in self.probs]
        lp += [-math.inf] * (8 - m)
        return _native.FAM["categorical"], lp[:4], lp[4:], m


@dataclass(frozen=True)
class Beta(Distribution):
    alpha: float
    beta: float

    family: ClassVar[str] = "beta"
    param_count: ClassVar[int] = 2

    def __post_init__(self):
        _check_positive("beta.alpha", self.alpha)
        _check_positive("beta.beta", self.beta)

    def params(self):
        return {"alpha": self.alpha, "beta": self.beta}

    def record(self):
        # distributions.py:404-409
        log_norm = log_gamma(self.alpha) + log_gamma(self.beta) - log_gamma(self.alpha + self.beta)
        return _rec("beta", [self.alpha, self.beta], [log_norm])


@dataclass(frozen=True)
class Weibull(Distribution):
    shape: float
    scale: float

    family: ClassVar[str] = "weibull"
    param_count: ClassVar[int] = 2

    def __post_init__(self):
        _check_positive("weibull.k", self.shape)
        _check_positive("weibull.lambda", self.scale)

    def params(self):
        return {"k": self.shape, "lambda": self.scale}

    def record(self):
        # distributions.py:427-435
        return _rec("weibull", [self.shape, self.scale], [math.log(self.shape) - math.log(self.scale)])


@dataclass(frozen=True)
class NegativeBinomial(Distribution):
    r: float
    p: float

    family: ClassVar[str] = "negative_binomial"
    param_count: ClassVar[int] = 2

    def __post_init__(self):
        _check_positive("negative_binomial.r", self.r)
        _check_finite("negative_binomial.p", self.p)
        if not (0.0 < self.p < 1.0):
            raise ValueError(f"negative_binomial.p must lie in (0, 1), got {self.p}")

    def params(self):
        return {"r": self.r, "p": self.p}

    def record(self):
        # distributions.py:455-465
        return _rec("negative_binomial", [self.r, self.p],
                    [log_gamma(self.r), self.r * math.log(self.p), math.log1p(-self.p)])


@dataclass(frozen=True)
class ChiSquared(Distribution):
    dof: float

    family: ClassVar[str] = "chi_squared"
    param_count: ClassVar[int] = 1

    def __post_init__(self):
        _check_positive("chi_squared.nu", self.dof)

    def params(self):
        return {"nu": self.dof}

    def record(self):
        # distributions.py:481-485
        half = self.dof / 2.0
        return _rec("chi_squared", [self.dof], [half * math.log(2.0), log_gamma(half), half - 1.0])


@dataclass(frozen=True)
class Pareto(Distribution):
    xm: float
    alpha: float

    family: ClassVar[str] = "pareto"
    param_count: ClassVar[int] = 2

    def __post_init__(self):
        _check_positive("pareto.xm", self.xm)
        _check_positive("pareto.alpha", self.alpha)

    def params(self):
        return {"xm": self.xm, "alpha": self.alpha}

    def record(self):
        # distributions.py:503-506
        c0 = math.log(self.alpha) + self.alpha * math.log(self.xm)
        return _rec("pareto", [self.xm, self.alpha], [c0, self.alpha + 1.0])


@dataclass(frozen=True)
class Joint(Distribution):
    """Factorised two-stream emission log p(y0, y1) = log p0(y0) + log p1(y1)
    (BASELINE config 4: Gamma step length + von Mises turning angle).  The
    reference API is 1-D only (inference.py:115); this record is the batched
    extension its oracle driver restates (oracle/loghmm_oracle.py)."""

    first: Distribution
    second: Distribution

    family: ClassVar[str] = "joint"

    def __post_init__(self):
        for d in (self.first, self.second):
            if isinstance(d, Joint) or not isinstance(d, Distribution):
                raise ValueError("joint emission takes two 1-D distributions")

    @property
    def param_count(self) -> int:  # type: ignore[override]
        return self.first.num_free_params() + self.second.num_free_params()

    def num_free_params(self) -> int:
        return self.param_count

    @property
    def n_streams(self) -> int:
        return 2

    def params(self):
        return {"first": self.first.params(), "second": self.second.params()}

    def record(self):
        raise TypeError("joint emissions are encoded per stream")


FAMILIES: dict[str, type[Distribution]] = {
    cls.family: cls
    for cls in (Gaussian, LogNormal, Exponential, Poisson, Rayleigh, Uniform, Categorical, VonMises,
                Gamma, Beta, Weibull, NegativeBinomial, ChiSquared, Pareto, StudentT)
}


def from_record(family: int, p: np.ndarray, aux: int = 0) -> Distribution:
    """Rebuild a record from device parameters (loghmm_mstep output)."""
    if family == _native.FAM["gaussian"]:
        return Gaussian(float(p[0]), float(p[1]))
    if family == _native.FAM["student_t"]:
        return StudentT(float(p[0]), float(p[1]), float(p[2]))
    if family == _native.FAM["gamma"]:
        return Gamma(float(p[0]), float(p[1]))
    if family == _native.FAM["von_mises"]:
        return VonMises(float(p[0]), float(p[1]))
    if family == _native.FAM["poisson"]:
        return Poisson(float(p[0]))
    name = _FAM_NAME.get(family)
    if name == "categorical":
        return Categorical(tuple(float(x) for x in p[: int(aux)]))
    if name in ("exponential", "rayleigh", "chi_squared"):
        return FAMILIES[name](float(p[0]))
    if name in FAMILIES:
        return FAMILIES[name](float(p[0]), float(p[1]))
    raise ValueError(f"unknown family id {family}")


_FAM_NAME = {v: k for k, v in _native.FAM.items()}
