"""Seeded synthetic inputs for the BASELINE.json configurations.

BASELINE.json names no public dataset; every config is a synthetic HMM draw
with the stated shapes and parameters.  Draw order (documented so the oracle
and the GPU see identical inputs): model parameters, then the state chain
(initial state, then one inverse-CDF draw per step for all sequences at
once), then the emissions.  All draws use ``np.random.default_rng(seed)``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .distributions import Gamma, Gaussian, Joint, Poisson, StudentT, VonMises
from .inference import HmmModel

__all__ = ["Config", "make_config", "CONFIGS", "sample_states"]


@dataclass
class Config:
    name: str
    B: int
    T: int
    K: int
    truth: HmmModel
    init: HmmModel | None
    data: np.ndarray  # [B, T] or [B, T, 2]
    msteps: int  # Baum-Welch M-steps of the full run (max_iterations = msteps + 1)


def sample_states(rng, pi, A, B, T):
    K = len(pi)
    cum_pi = np.cumsum(pi)
    cumA = np.cumsum(A, axis=1)
    s = np.empty((B, T), dtype=np.int64)
    s[:, 0] = np.minimum(np.searchsorted(cum_pi, rng.random(B), side="right"), K - 1)
    for t in range(1, T):
        u = rng.random(B)
        s[:, t] = np.minimum((u[:, None] >= cumA[s[:, t - 1]]).sum(axis=1), K - 1)
    return s


def _sticky(diag):
    K = len(diag)
    A = np.empty((K, K))
    for i, d in enumerate(diag):
        A[i] = (1.0 - d) / (K - 1)
        A[i, i] = d
    return A


def make_config(name: str, B: int | None = None, T: int | None = None, seed: int = 0) -> Config:
    rng = np.random.default_rng(seed)
    if name == "c1":
        B, T = B or 1, T or 1000
        pi = np.array([0.5, 0.5])
        A = np.array([[0.95, 0.05], [0.10, 0.90]])
        mu, sd = np.array([-1.0, 2.0]), np.array([0.7, 1.2])
        truth = HmmModel(pi, A, tuple(Gaussian(float(m), float(s)) for m, s in zip(mu, sd)))
        s = sample_states(rng, pi, A, B, T)
        y = mu[s] + sd[s] * rng.standard_normal((B, T))
        init = HmmModel([0.5, 0.5], [[0.9, 0.1], [0.1, 0.9]], (Gaussian(-0.5, 1.0), Gaussian(1.5, 1.0)))
        return Config(name, B, T, 2, truth, init, y, 1)
    if name == "c2":
        B, T, K = B or 4096, T or 1024, 4
        pi = np.full(K, 1.0 / K)
        A = 0.1 * rng.dirichlet(np.ones(K), size=K) + 0.9 * np.eye(K)
        A = A / A.sum(axis=1, keepdims=True)
        mu = np.array([-3.0, -1.0, 1.0, 3.0])
        sd = rng.uniform(0.5, 1.5, K)
        truth = HmmModel(pi, A, tuple(Gaussian(float(m), float(s)) for m, s in zip(mu, sd)))
        s = sample_states(rng, pi, A, B, T)
        y = mu[s] + sd[s] * rng.standard_normal((B, T))
        mu0 = mu + rng.normal(0.0, 0.3, K)
        init = HmmModel(pi, A, tuple(Gaussian(float(m), float(v * 1.2)) for m, v in zip(mu0, sd)))
        return Config(name, B, T, K, truth, init, y, 10)
    if name == "c3":
        B, T, K = B or 1024, T or 2048, 3
        pi = np.full(K, 1.0 / K)
        A = _sticky([0.97, 0.95, 0.90])
        mu, sd, nu = np.array([-0.02, 0.0, 0.02]), np.array([0.005, 0.01, 0.03]), np.array([3.0, 5.0, 10.0])
        truth = HmmModel(pi, A, tuple(StudentT(*map(float, p)) for p in zip(mu, sd, nu)))
        s = sample_states(rng, pi, A, B, T)
        y = mu[s] + sd[s] * rng.standard_t(nu[s])
        init = HmmModel(pi, A, tuple(StudentT(float(m) * 0.5, float(v) * 1.3, 8.0) for m, v in zip(mu, sd)))
        return Config(name, B, T, K, truth, init, y, 20)
    if name == "c4":
        B, T, K = B or 2048, T or 2000, 3
        pi = np.full(K, 1.0 / K)
        A = _sticky([0.85, 0.80, 0.90])
        shape, scale = np.array([0.8, 2.0, 5.0]), np.array([0.1, 0.5, 1.5])
        vmu, kap = np.array([math.pi, 0.0, 0.0]), np.array([0.5, 2.0, 8.0])
        truth = HmmModel(pi, A, tuple(
            Joint(Gamma(float(a), float(1.0 / b)), VonMises(float(m), float(k)))
            for a, b, m, k in zip(shape, scale, vmu, kap)))
        s = sample_states(rng, pi, A, B, T)
        step = rng.gamma(shape[s], scale[s])
        ang = rng.vonmises(vmu[s], kap[s])
        ang = np.where(ang <= -math.pi, ang + 2 * math.pi, ang)
        y = np.stack([step, ang], axis=-1)
        init = HmmModel(pi, A, tuple(
            Joint(Gamma(float(a) * 1.1, float(0.9 / b)), VonMises(float(m) - 0.1 if m > 0 else 0.1, float(k) * 0.8))
            for a, b, m, k in zip(shape, scale, vmu, kap)))
        return Config(name, B, T, K, truth, init, y, 20)
    if name == "c5":
        B, T, K = B or 64, T or 65536, 64
        pi = np.full(K, 1.0 / K)
        A = np.zeros((K, K))
        for i in range(K):
            nb = [j for j in range(max(0, i - 4), min(K, i + 5)) if j != i]
            A[i, nb] = 0.2 * rng.dirichlet(np.ones(len(nb)))
            A[i, i] = 0.8
        A = A / A.sum(axis=1, keepdims=True)
        lam = 0.5 * (np.arange(K) + 1.0)
        truth = HmmModel(pi, A, tuple(Poisson(float(l)) for l in lam))
        s = sample_states(rng, pi, A, B, T)
        y = rng.poisson(lam[s]).astype(np.float64)
        init = HmmModel(pi, A, tuple(Poisson(float(l) * 1.1) for l in lam))
        return Config(name, B, T, K, truth, init, y, 5)
    raise ValueError(name)


CONFIGS = ("c1", "c2", "c3", "c4", "c5")
