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

Families outside the hot path (LogNormal, Exponential, Rayleigh, Uniform,
Categorical, Beta, Weibull, NegativeBinomial, ChiSquared, Pareto;
SURVEY.md §8f item 2) are not provided.
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
    cls.family: cls for cls in (Gaussian, Poisson, VonMises, Gamma, StudentT)
}


def from_record(family: int, p: np.ndarray) -> Distribution:
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
    raise ValueError(f"unknown family id {family}")
