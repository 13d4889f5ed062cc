#!/usr/bin/env python3
"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the unmodified reference package read-only from
/root/reference/pkg/src (no bytecode written) and freezes:

  frontend.json   the reference's own frozen binding fixtures
                  (pkg/frontend/fixtures/{earthquake,small_models}.json,
                  made by pkg/scripts/make_binding_fixtures.py), re-emitted
                  for the hot-path families (categorical case dropped);
  vectors.npz     per-case inputs and the reference's outputs for seeded
                  small models of every hot-path family: emission matrix,
                  log_alpha, log_beta, gamma, xi, LL, Viterbi path and
                  log_joint, and a short Baum-Welch run (trace + params);
  cases.json      the case index (model parameters per case).

The GPU box never reads /root/reference; tests read only these files.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from loghmm.distributions import Gamma, Gaussian, Poisson, StudentT, VonMises  # noqa: E402
from loghmm.inference import HmmModel, emission_log_matrix, posteriors, viterbi  # noqa: E402
from loghmm.training import TrainingConfig, baum_welch  # noqa: E402

OUT = Path(__file__).resolve().parent


def fam_tuple(d):
    if isinstance(d, Gaussian):
        return ["gaussian", d.mu, d.sigma]
    if isinstance(d, StudentT):
        return ["student_t", d.mu, d.sigma, d.nu]
    if isinstance(d, Gamma):
        return ["gamma", d.shape, d.rate]
    if isinstance(d, VonMises):
        return ["von_mises", d.mu, d.kappa]
    if isinstance(d, Poisson):
        return ["poisson", d.rate]
    raise TypeError(d)


def random_model(rng, family, k):
    pi = rng.dirichlet(np.ones(k))
    a = rng.dirichlet(np.ones(k), size=k) * 0.5 + 0.5 * np.eye(k)
    a = a / a.sum(axis=1, keepdims=True)
    if family == "gaussian":
        em = [Gaussian(float(rng.normal(0, 2)), float(rng.uniform(0.4, 1.6))) for _ in range(k)]
        sample = lambda s: rng.normal([e.mu for e in em], [e.sigma for e in em])[s]  # noqa: E731
    elif family == "student_t":
        em = [StudentT(float(rng.normal(0, 1)), float(rng.uniform(0.3, 1.2)), float(rng.uniform(2.5, 12))) for _ in range(k)]
        sample = lambda s: np.array([em[i].mu + em[i].sigma * rng.standard_t(em[i].nu) for i in s])  # noqa: E731
    elif family == "gamma":
        em = [Gamma(float(rng.uniform(0.7, 5)), float(rng.uniform(0.5, 3))) for _ in range(k)]
        sample = lambda s: np.array([rng.gamma(em[i].shape, 1.0 / em[i].rate) for i in s])  # noqa: E731
    elif family == "von_mises":
        em = [VonMises(float(rng.uniform(-3, 3)), float(rng.uniform(0.3, 6))) for _ in range(k)]
        sample = lambda s: np.array([rng.vonmises(em[i].mu, em[i].kappa) for i in s])  # noqa: E731
    elif family == "poisson":
        em = [Poisson(float(rng.uniform(0.5, 12))) for _ in range(k)]
        sample = lambda s: np.array([rng.poisson(em[i].rate) for i in s], dtype=float)  # noqa: E731
    else:
        raise ValueError(family)
    return HmmModel(pi, a, tuple(em)), sample


def draw_states(rng, model, T):
    s = [int(rng.choice(model.num_states, p=model.initial))]
    for _ in range(T - 1):
        s.append(int(rng.choice(model.num_states, p=model.transitions[s[-1]])))
    return np.array(s)


def main():
    # -- frontend fixtures -------------------------------------------------
    eq = json.loads((REF / "frontend/fixtures/earthquake.json").read_text())
    small = json.loads((REF / "frontend/fixtures/small_models.json").read_text())
    front = {"earthquake": eq, "small_models": [c for c in small if c["name"] != "discrete-2"]}
    (OUT / "frontend.json").write_text(json.dumps(front, indent=1) + "\n")

    # -- seeded per-family cases -------------------------------------------
    rng = np.random.default_rng(20261019)
    arrays = {}
    cases = []
    plan = []
    for fam in ("gaussian", "student_t", "gamma", "von_mises", "poisson"):
        for k, T in ((2, 60), (3, 150), (4, 97)):
            plan.append((fam, k, T))
    plan.append(("gaussian", 1, 25))
    plan.append(("gaussian", 4, 1))
    for idx, (fam, k, T) in enumerate(plan):
        model, sample = random_model(rng, fam, k)
        y = sample(draw_states(rng, model, T)).astype(float)
        fb = posteriors(model, y, include_xi=True)
        vit = viterbi(model, y)
        cfg = TrainingConfig(max_iterations=3, rel_tol=1e-300)
        fitted, rep = baum_welch(model, [y, y[::-1].copy()], cfg)
        name = f"case{idx:02d}"
        arrays[f"{name}_y"] = y
        arrays[f"{name}_logb"] = emission_log_matrix(model, y)
        arrays[f"{name}_log_alpha"] = fb.log_alpha
        arrays[f"{name}_log_beta"] = fb.log_beta
        arrays[f"{name}_gamma"] = fb.gamma
        arrays[f"{name}_xi"] = fb.xi
        arrays[f"{name}_path"] = vit.path
        arrays[f"{name}_bw_pi"] = fitted.initial
        arrays[f"{name}_bw_A"] = fitted.transitions
        cases.append({
            "name": name, "family": fam, "K": k, "T": T,
            "pi": model.initial.tolist(), "A": model.transitions.tolist(),
            "emissions": [fam_tuple(d) for d in model.emissions],
            "ll": fb.log_likelihood, "log_joint": vit.log_joint,
            "bw": {"max_iterations": 3, "trace": rep.log_likelihood_trace,
                   "emissions": [fam_tuple(d) for d in fitted.emissions],
                   "collapsed": rep.collapsed_states},
        })

    # -- config 1 (BASELINE.json configs[0]) ---------------------------------
    sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
    c1_rng = np.random.default_rng(0)
    pi = np.array([0.5, 0.5])
    A = np.array([[0.95, 0.05], [0.10, 0.90]])
    mu, sd = np.array([-1.0, 2.0]), np.array([0.7, 1.2])
    # identical draw order to paper_2605_29208_b200/configs.py (c1)
    cum_pi, cumA = np.cumsum(pi), np.cumsum(A, axis=1)
    s = np.empty((1, 1000), dtype=np.int64)
    s[:, 0] = np.minimum(np.searchsorted(cum_pi, c1_rng.random(1), side="right"), 1)
    for t in range(1, 1000):
        u = c1_rng.random(1)
        s[:, t] = np.minimum((u[:, None] >= cumA[s[:, t - 1]]).sum(axis=1), 1)
    y = (mu[s] + sd[s] * c1_rng.standard_normal((1, 1000)))[0]
    truth = HmmModel(pi, A, (Gaussian(-1.0, 0.7), Gaussian(2.0, 1.2)))
    init = HmmModel([0.5, 0.5], [[0.9, 0.1], [0.1, 0.9]], (Gaussian(-0.5, 1.0), Gaussian(1.5, 1.0)))
    fb = posteriors(init, y)
    vit = viterbi(init, y)
    fitted, rep = baum_welch(init, [y], TrainingConfig(max_iterations=2, rel_tol=1e-300))
    arrays["c1_y"] = y
    arrays["c1_log_alpha"] = fb.log_alpha
    arrays["c1_log_beta"] = fb.log_beta
    arrays["c1_gamma"] = fb.gamma
    arrays["c1_path"] = vit.path
    arrays["c1_truth_path"] = viterbi(truth, y).path
    c1 = {"ll": fb.log_likelihood, "log_joint": vit.log_joint,
          "bw_trace": rep.log_likelihood_trace,
          "bw_pi": fitted.initial.tolist(), "bw_A": fitted.transitions.tolist(),
          "bw_emissions": [fam_tuple(d) for d in fitted.emissions]}

    # -- T = 100000 underflow case (test_acceptance.py:94-105) ---------------
    urng = np.random.default_rng(7)
    umodel = HmmModel([0.5, 0.5], [[0.97, 0.03], [0.05, 0.95]], (Gaussian(0.0, 1.0), Gaussian(2.5, 1.8)))
    useq = urng.normal(size=100_000) * 2.0 + 1.0
    ufb = posteriors(umodel, useq)
    under = {"ll": ufb.log_likelihood, "gamma_row0": ufb.gamma[0].tolist(),
             "gamma_last": ufb.gamma[-1].tolist(), "viterbi_log_joint": viterbi(umodel, useq).log_joint}

    np.savez_compressed(OUT / "vectors.npz", **arrays)
    (OUT / "cases.json").write_text(json.dumps({"cases": cases, "c1": c1, "underflow": under}, indent=1) + "\n")
    print(f"wrote {len(cases)} cases + c1 + underflow to {OUT}")


if __name__ == "__main__":
    main()
