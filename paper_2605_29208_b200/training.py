"""Drop-in for the reference training layer (training.py), on B200.

Baum-Welch keeps the reference's control flow and semantics
(training.py:160-236): the trace holds the log-likelihood at the start of
each iteration, convergence is |delta| < rel_tol*|LL| (or delta == 0), and the
last iteration applies no M-step, so ``max_iterations=N`` runs N E-steps and
N-1 M-steps.  Each E-step is one fused kernel over the whole batch
(loghmm_forward_backward with statistics) plus a deterministic reduction;
each M-step is one per-state kernel (loghmm_mstep) and, for Student-t
states, the ECME likelihood-guard pass.  The model stays on the device
between iterations; the host reads back only per-sequence flags and
likelihoods (for the reference's error semantics) and the per-state status.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native, engine
from .distributions import (
    SCALE_FLOOR,
    VONMISES_KAPPA_CEILING,
    Distribution,
    EcmeConfig,
    FitWarning,
    Gamma,
    Gaussian,
    Joint,
    Poisson,
    StudentT,
    VonMises,
    from_record,
)
from .inference import HmmModel

__all__ = [
    "TrainingConfig",
    "TrainingReport",
    "TrainingError",
    "ModelScore",
    "baum_welch",
    "score_model",
    "count_parameters",
    "default_initial_model",
]


class TrainingError(ValueError):
    """Raised when the data cannot be trained under the requested model."""


@dataclass(frozen=True)
class TrainingConfig:
    """EM control knobs; defaults favor convergence over speed (training.py:46-61)."""

    max_iterations: int = 500
    rel_tol: float = 1e-8
    collapse_epsilon: float = 1e-8
    ecme: EcmeConfig = field(default_factory=EcmeConfig)

    def __post_init__(self):
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be positive")
        if not (0.0 < self.rel_tol < 1.0):
            raise ValueError("rel_tol must lie in (0, 1)")
        if self.collapse_epsilon <= 0.0:
            raise ValueError("collapse_epsilon must be positive")


@dataclass
class TrainingReport:
    log_likelihood_trace: list[float]
    iterations: int
    converged: bool
    collapsed_states: list[tuple[int, int]]


@dataclass(frozen=True)
class ModelScore:
    log_likelihood: float
    num_params: int
    num_obs: int
    aic: float
    bic: float
    aicc: float | None


def count_parameters(model: HmmModel) -> int:
    """training.py:82-86."""
    k = model.num_states
    return (k - 1) + k * (k - 1) + sum(d.num_free_params() for d in model.emissions)


_FAM_NAME = {v: k for k, v in _native.FAM.items()}

_SUPPORT_TEXT = {  # distributions.py:623-629 _validate_support and the per-fit checks
    "poisson": "poisson fit requires non-negative integer observations",
    "gamma": "gamma fit requires strictly positive observations",
    "lognormal": "lognormal fit requires strictly positive observations",
    "exponential": "exponential fit requires non-negative observations",
    "rayleigh": "rayleigh fit requires non-negative observations",
    "categorical": "categorical fit requires non-negative integer observations",
    "beta": "beta fit requires observations strictly inside (0, 1)",
    "weibull": "weibull fit requires strictly positive observations",
    "negative_binomial": "negative_binomial fit requires non-negative integer observations",
    "chi_squared": "chi_squared fit requires strictly positive observations",
    "pareto": "pareto fit requires strictly positive observations",
}
_DEGENERATE_TEXT = {
    "exponential": "exponential fit is degenerate: weighted mean is zero",
    "weibull": "weibull fit is degenerate: weighted variance is zero",
    "negative_binomial": "negative_binomial fit is degenerate: all observations are zero",
    "pareto": "pareto fit is degenerate: all weighted observations equal the minimum",
}

_ERR_TEXT = {
    _native.MS_ERR_NO_MASS: lambda fam: "fit requires positive total weight",
    _native.MS_ERR_SUPPORT: lambda fam: _SUPPORT_TEXT.get(fam, f"{fam} fit support violation"),
    _native.MS_ERR_DEGENERATE: lambda fam: _DEGENERATE_TEXT.get(fam, f"{fam} fit is degenerate"),
    _native.MS_ERR_GAMMA_VAR: lambda fam: "gamma fit is degenerate: weighted variance is zero",
    _native.MS_ERR_GAMMA_GAP: lambda fam: "gamma fit is degenerate: zero log-moment gap",
    _native.MS_ERR_NONFINITE: lambda fam: "von_mises fit requires finite angles",
}


def _warn_texts(fam: str, st: int) -> list[str]:
    out = []
    if fam == "gamma" and st & _native.MS_WARN_NEWTON:
        out.append("gamma shape update did not converge; using moment seed")
    if fam == "von_mises":
        if st & _native.MS_WARN_BOUNDARY:
            out.append("von_mises resultant length is at the boundary; clamping concentration")
        if st & _native.MS_WARN_CEILING:
            out.append("von_mises concentration clamped at ceiling")
        if st & _native.MS_WARN_NEWTON:
            out.append("von_mises concentration update did not converge")
    if fam == "student_t" and st & _native.MS_WARN_CEILING:
        out.append("student_t degrees of freedom clamped; near-Gaussian state")
    if fam == "beta" and st & _native.MS_WARN_ITERCAP:
        out.append("beta fit hit the iteration cap before tolerance")
    if fam == "weibull" and st & _native.MS_WARN_NEWTON:
        out.append("weibull shape update did not converge; using moment seed")
    if fam == "chi_squared" and st & _native.MS_WARN_NEWTON:
        out.append("chi_squared update did not converge; using mean seed")
    if fam == "negative_binomial":
        if st & _native.MS_WARN_BOUNDARY:
            out.append("negative_binomial data is underdispersed; returning near-Poisson boundary fit")
        if st & _native.MS_WARN_CEILING:
            out.append("negative_binomial dispersion clamped; data is near-Poisson")
        if st & _native.MS_WARN_NEWTON:
            out.append("negative_binomial dispersion update did not converge")
    return out


def _natural(em) -> np.ndarray:
    """Natural parameters of a device record (categorical keeps log p_k in
    its 8 slots: p = exp(log p)))."""
    if int(em["family"]) == _native.FAM["categorical"]:
        m = int(em["reserved"])
        return np.exp(np.concatenate([em["p"], em["c"]]))[:m]
    return em["p"]


def apply_mstep_status(st: np.ndarray, fams, stacklevel: int = 2, cats=None) -> list[int]:
    """Raise / warn for the per-state M-step status words the way
    m_step_emissions and the family fits do (training.py:130-148,
    distributions.py FitWarning sites); returns the collapsed states.

    ``fams[s][j]`` is the family code of state j in stream s."""
    ns = len(fams)
    K = len(fams[0])
    collapsed = []
    for j in range(K):
        for s in range(ns):
            code = int(st[s * K + j])
            fam = _FAM_NAME[fams[s][j]]
            base = code & 0xFF
            if base == _native.MS_ERR_CAT_CODE:
                m = int(cats[s][j]) if cats is not None else 0
                raise TrainingError(f"state {j}: categorical fit saw code >= {m}")
            if base >= 16:
                raise TrainingError(f"state {j}: {_ERR_TEXT[base](fam)}")
            for msg in _warn_texts(fam, code):
                warnings.warn(msg, FitWarning, stacklevel=stacklevel)
        if int(st[j]) & 0xFF == _native.MS_COLLAPSED:
            collapsed.append(j)
    return collapsed


def model_from_record(rec: np.ndarray, keep=None) -> HmmModel:
    """HmmModel from a device loghmm_model_t read back to the host.  States
    whose ``keep[j]`` is not None return that object (collapsed states keep
    their distribution object, training.py:139-141)."""
    K = int(rec["K"])
    ns = int(rec["n_streams"])
    ems = []
    for j in range(K):
        if keep is not None and keep[j] is not None:
            ems.append(keep[j])
            continue
        parts = [from_record(int(rec["em"][s, j]["family"]), _natural(rec["em"][s, j]),
                             int(rec["em"][s, j]["reserved"])) for s in range(ns)]
        ems.append(parts[0] if ns == 1 else Joint(parts[0], parts[1]))
    pi = np.array(rec["pi"][:K], dtype=float)
    A = np.array(rec["A"][: K * K], dtype=float).reshape(K, K)
    return HmmModel(pi, A, tuple(ems))


def _check_estep(flags: np.ndarray, ll: np.ndarray) -> None:
    """Reference error order: NaN at validation, then per sequence the dead
    observation check (training.py:189-194) and the -inf LL check (:196-197)."""
    if (flags[:, 1] & 1).any():
        raise ValueError("observation sequence contains NaN")
    bad = np.nonzero((flags[:, 0] >= 0) | (ll == -np.inf))[0]
    if bad.size:
        s = int(bad[0])
        if flags[s, 0] >= 0:
            raise TrainingError(
                "observation outside the support of every state: "
                f"sequence {s}, index {int(flags[s, 0])}"
            )
        raise TrainingError(f"sequence {s} is impossible under the model")
    rng = np.nonzero(flags[:, 1] & 4)[0]
    if rng.size:
        from .inference import RANGE_MSG

        raise FloatingPointError(RANGE_MSG.format(s=int(rng[0])))


def baum_welch(model: HmmModel, data, config: TrainingConfig | None = None, dtype="float64"):
    """EM training: returns the refined model and the per-iteration trace."""
    config = config or TrainingConfig()
    ns = model.n_streams
    if isinstance(data, (list, tuple)) and len(data) == 0:
        raise TrainingError("training data contains no sequences")  # training.py:151-156
    batch = engine.make_batch(data, ns, dtype)
    K = model.num_states
    dm_cur = engine.DeviceModel.from_model(model)
    dm_next = engine.DeviceModel.empty_like(dm_cur)
    fams = [[int(dm_cur.host["em"][s, j]["family"]) for j in range(K)] for s in range(ns)]
    student = [(s, j) for s in range(ns) for j in range(K) if fams[s][j] == _native.FAM["student_t"]]
    student_streams = sorted({s for s, _ in student})
    var_fams = (_native.FAM["gaussian"], _native.FAM["gamma"], _native.FAM["student_t"])
    var_streams = [s for s in range(ns) if any(f in var_fams for f in fams[s])]
    ext_streams = [s for s in range(ns) if any(f >= _native.FAM["lognormal"] for f in fams[s])]
    cats = [[int(dm_cur.host["em"][s, j]["reserved"]) for j in range(K)] for s in range(ns)]
    dev = batch.y0.device
    # gamma is materialised for the exact second passes (variance, ECME guard)
    # and the weighted-sample fits of the families 6..15
    need_gamma = bool(student) or bool(var_streams) or bool(ext_streams)
    out = engine.forward_backward(batch, dm_cur, alpha=False, beta=False, gamma=need_gamma,
                                  stats=True)
    totals = torch.empty(out.partials.shape[1] + 1, dtype=torch.float64, device=dev)
    status = torch.zeros(ns * K, dtype=torch.int32, device=dev)
    guard = torch.zeros(ns * K * engine.GUARD_STRIDE, dtype=torch.float64, device=dev)
    need_more = torch.zeros(1, dtype=torch.int32, device=dev)

    trace: list[float] = []
    collapsed_states: list[tuple[int, int]] = []
    converged = False
    n_msteps = 0
    kept = list(model.emissions)  # objects untouched by every M-step so far
    for iteration in range(1, config.max_iterations + 1):
        if iteration > 1:
            engine.forward_backward(batch, dm_cur, alpha=False, beta=False, gamma=need_gamma,
                                    stats=True, out=out)
        engine.reduce_stats(out.partials, out.ll, totals)
        flags = out.flags.cpu().numpy()
        ll = out.ll.cpu().numpy()
        _check_estep(flags, ll)
        total_ll = float(totals[-1].item())
        trace.append(total_ll)
        if len(trace) >= 2:
            delta = trace[-1] - trace[-2]
            if delta == 0.0 or abs(delta) < config.rel_tol * abs(trace[-1]):
                converged = True
                break
        if iteration == config.max_iterations:
            break
        engine.mstep(dm_cur, totals, batch.B, config, dm_next, status, guard, batch.dtype)
        for s in var_streams:
            engine.variance_pass(batch, dm_next, out.gamma, s, guard, status)
        for s in student_streams:
            ncand = 2
            while True:
                need_more.zero_()
                engine.student_guard(batch, dm_next, out.gamma, s, ncand, guard, status, need_more)
                if int(need_more.item()) == 0:
                    break
                ncand = _native.GUARD_CANDIDATES
        for s in ext_streams:
            engine.ext_fit(batch, dm_next, out.gamma, s, guard, status, need_more)
        collapsed = apply_mstep_status(status.cpu().numpy(), fams, stacklevel=3, cats=cats)
        collapsed_states.extend((iteration, j) for j in collapsed)
        # a collapsed state keeps its distribution object (m_step_emissions
        # returns ``dist`` itself, training.py:139-141)
        for j in range(K):
            if j not in collapsed:
                kept[j] = None
        dm_cur, dm_next = dm_next, dm_cur
        n_msteps += 1

    current = model if n_msteps == 0 else model_from_record(dm_cur.to_host(), keep=kept)
    report = TrainingReport(
        log_likelihood_trace=trace,
        iterations=len(trace),
        converged=converged,
        collapsed_states=collapsed_states,
    )
    return current, report


def score_model(model: HmmModel, data, dtype="float64") -> ModelScore:
    """Log-likelihood over all sequences plus AIC/BIC/AICc (training.py:89-102)."""
    batch = engine.make_batch(data, model.n_streams, dtype)
    dm = engine.DeviceModel.from_model(model)
    o = engine.forward_backward(batch, dm, alpha=False, beta=False, gamma=False)
    flags = o.flags.cpu().numpy()
    if (flags[:, 1] & 1).any():
        raise ValueError("observation sequence contains NaN")
    total_ll = float(np.sum(o.ll.cpu().numpy()))
    n = batch.N
    p = count_parameters(model)
    aic = 2.0 * p - 2.0 * total_ll
    bic = p * math.log(n) - 2.0 * total_ll
    aicc = aic + 2.0 * p * (p + 1.0) / (n - p - 1.0) if n > p + 1 else None
    return ModelScore(total_ll, p, n, aic, bic, aicc)


# ---------------------------------------------------------------------------
# default_initial_model on the device (training.py:239-282)
# ---------------------------------------------------------------------------
_SUPPORT_SEED = {  # distributions.py:623-629 texts raised by moment_seed
    "positive": "{} fit requires strictly positive observations",
    "unit": "{} fit requires observations strictly inside (0, 1)",
    "integer": "{} fit requires non-negative integer observations",
}


def _seed_from_moments(family: str, row: np.ndarray, pool: np.ndarray, num_categories) -> Distribution:
    """moment_seed (distributions.py:1130-1176) from one bin's device
    moments (loghmm_bin_moments row; ``pool`` = the row of the whole pool,
    used by uniform / pareto, whose M-steps pin the global range)."""
    from .distributions import (
        NEGBINOM_R_CEILING, Beta, Categorical, ChiSquared, Exponential, LogNormal, NegativeBinomial,
        Pareto, Rayleigh, Uniform, Weibull)

    n, mean, var = float(row[0]), float(row[1]), float(row[2])
    sd = max(math.sqrt(var), SCALE_FLOOR)

    def need(kind, bad):
        if bad > 0:
            raise ValueError(_SUPPORT_SEED[kind].format(family))

    if family == "gaussian":
        return Gaussian(mean, sd)
    if family == "lognormal":
        need("positive", row[10])
        return LogNormal(float(row[3]), max(math.sqrt(float(row[4])), SCALE_FLOOR))
    if family == "exponential":
        return Exponential(1.0 / max(mean, SCALE_FLOOR))
    if family == "poisson":
        return Poisson(max(mean, SCALE_FLOOR))
    if family == "rayleigh":
        return Rayleigh(max(math.sqrt(float(row[7]) / (2.0 * n)), SCALE_FLOOR))
    if family == "uniform":  # fit_uniform on the pool (distributions.py:676-684)
        lo, hi = float(pool[8]), float(pool[9])
        if hi <= lo:
            hi = lo + SCALE_FLOOR
        return Uniform(lo, hi)
    if family == "categorical":  # fit_categorical (distributions.py:687-699)
        need("integer", row[13])
        if num_categories > 8:
            raise ValueError(f"categorical with {num_categories} categories: the device record holds at most 8")
        counts = np.asarray(row[14:14 + num_categories], dtype=float)
        probs = counts / n
        probs = probs / probs.sum()
        return Categorical(tuple(float(p) for p in probs))
    if family == "von_mises":
        s_, c_ = float(row[5]), float(row[6])
        mu = math.atan2(s_, c_)
        if mu <= -math.pi:
            mu = math.pi
        rbar = min(math.hypot(s_, c_) / n, 1.0 - 1e-9)
        kappa = rbar * (2.0 - rbar * rbar) / (1.0 - rbar * rbar)
        return VonMises(mu, min(kappa, VONMISES_KAPPA_CEILING))
    if family == "gamma":
        need("positive", row[10])
        shape = mean * mean / var if var > 0 else 1.0
        return Gamma(max(shape, SCALE_FLOOR), max(shape, SCALE_FLOOR) / max(mean, SCALE_FLOOR))
    if family == "beta":
        need("unit", row[12])
        scale = mean * (1.0 - mean) / var - 1.0 if var > 0 else -1.0
        if scale <= 0:
            return Beta(1.0, 1.0)
        return Beta(mean * scale, (1.0 - mean) * scale)
    if family == "weibull":
        need("positive", row[10])
        k = (mean / sd) ** 1.086 if var > 0 else 1.0
        scale = mean / math.exp(math.lgamma(1.0 + 1.0 / k))
        return Weibull(k, max(scale, SCALE_FLOOR))
    if family == "negative_binomial":
        need("integer", row[13])
        if mean <= 0:
            raise ValueError("negative_binomial seed is degenerate: zero mean")
        r = mean * mean / (var - mean) if var > mean else NEGBINOM_R_CEILING
        return NegativeBinomial(r, r / (r + mean))
    if family == "chi_squared":
        need("positive", row[10])
        return ChiSquared(max(mean, SCALE_FLOOR))
    if family == "pareto":  # fit_pareto on the pool (distributions.py:702-710)
        need("positive", pool[10])
        npool, xm = float(pool[0]), float(pool[8])
        denom = npool * (float(pool[3]) - math.log(xm))
        if denom <= 0.0:
            raise ValueError("pareto fit is degenerate: all weighted observations equal the minimum")
        return Pareto(xm, npool / denom)
    if family == "student_t":
        return StudentT(mean, sd, 10.0)
    raise ValueError(f"unknown family '{family}'")


def default_initial_model(num_states: int, families, data) -> HmmModel:
    """Deterministic starting model: pooled observations sorted and split into
    quantile bins, one per state, each seeded from its bin's moments; uniform
    start with sticky diagonals (training.py:239-282).  The pool is sorted on
    the device and loghmm_bin_moments reduces every bin in one launch; only
    K rows of moments come back to the host."""
    if num_states < 1:
        raise ValueError("num_states must be positive")
    if isinstance(families, str):
        families = [families]
    families = list(families)
    if len(families) == 1:
        families = families * num_states
    if len(families) != num_states:
        raise ValueError(f"expected 1 or {num_states} family names, got {len(families)}")
    if isinstance(data, (list, tuple)) and len(data) == 0:
        raise TrainingError("training data contains no sequences")
    batch = engine.make_batch(data, 1, "float64")
    if bool(torch.isnan(batch.y0).any()):
        raise ValueError("observation sequence contains NaN")
    N = batch.N
    if N < num_states:
        raise TrainingError("more states than observations; cannot seed bins")
    pooled = torch.sort(batch.y0).values  # device radix sort (np.sort of the pool)
    L = _native.lib()
    rows = torch.empty((num_states, _native.BIN_SLOTS), dtype=torch.float64, device=pooled.device)
    _native.check(L.loghmm_bin_moments(pooled.data_ptr(), N, num_states, rows.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream), "loghmm_bin_moments")
    pool = torch.empty((1, _native.BIN_SLOTS), dtype=torch.float64, device=pooled.device)
    _native.check(L.loghmm_bin_moments(pooled.data_ptr(), N, 1, pool.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream), "loghmm_bin_moments")
    rows, pool = rows.cpu().numpy(), pool.cpu().numpy()[0]
    num_categories = int(pool[9]) + 1 if "categorical" in families else None
    emissions = [_seed_from_moments(f, rows[j], pool, num_categories) for j, f in enumerate(families)]
    pi = np.full(num_states, 1.0 / num_states)
    if num_states == 1:
        a = np.array([[1.0]])
    else:
        off = 0.1 / (num_states - 1)
        a = np.full((num_states, num_states), off)
        np.fill_diagonal(a, 0.9)
    return HmmModel(pi, a, tuple(emissions))
