"""CPU oracle for the log-space HMM hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm
(/root/reference/pkg/src/loghmm, Python/numpy, fp64).  It is imported only by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg, always as the checker or the CPU baseline, never as the product path.

Pinning: tests/test_oracle_golden.py checks it against
  * the reference's own frozen fixtures (frontend/fixtures/*.json, re-emitted
    into tests/golden/ by tests/golden/make_golden.py), and
  * golden vectors produced by importing the reference itself in the build
    container (same script), bit-exact where the reference uses only IEEE
    basic operations (Gaussian / Poisson emissions, Viterbi), <=1e-12 else.

Each function cites the reference file:line it restates.  fp32 variants
(``dtype=np.float32``) restate the same operation order in float32; the
reference has no fp32 path (it forces float64, inference.py:114), so these
define the fp32 contract.
"""

from __future__ import annotations

import math
import warnings

import numpy as np

LOG_2PI = math.log(2.0 * math.pi)
SCALE_FLOOR = 1e-9
KAPPA_CEIL = 1e5

# ----------------------------------------------------------------------------
# special functions (special.py)
# ----------------------------------------------------------------------------


def lse_axis(a: np.ndarray, axis: int) -> np.ndarray:
    """special.py:48-62: max-shifted log-sum-exp; all -inf -> -inf."""
    mx = np.max(a, axis=axis, keepdims=True)
    ok = np.isfinite(mx)
    sh = np.where(ok, a - np.where(ok, mx, 0.0), -np.inf)
    with np.errstate(divide="ignore"):
        return np.log(np.sum(np.exp(sh), axis=axis)) + np.squeeze(np.where(ok, mx, -np.inf), axis=axis)


def digamma(x: float) -> float:
    """special.py:81-103."""
    acc = 0.0
    while x < 10.0:
        acc -= 1.0 / x
        x += 1.0
    r = 1.0 / x
    r2 = r * r
    tail = 1.0 / 12.0 - r2 * (1.0 / 120.0 - r2 * (1.0 / 252.0 - r2 * (1.0 / 240.0 - r2 / 132.0)))
    return acc + (math.log(x) - 0.5 * r - r2 * tail)


def trigamma(x: float) -> float:
    """special.py:106-128."""
    acc = 0.0
    while x < 10.0:
        acc += 1.0 / (x * x)
        x += 1.0
    r = 1.0 / x
    r2 = r * r
    inner = 1.0 / 30.0 - r2 * (1.0 / 42.0 - r2 * (1.0 / 30.0 - 5.0 * r2 / 66.0))
    return acc + r * (1.0 + r * (0.5 + r * (1.0 / 6.0 - r2 * inner)))


_I0S = (1.0, 3.5156229, 3.0899424, 1.2067492, 0.2659732, 0.0360768, 0.0045813)
_I0L = (0.39894228, 0.01328592, 0.00225319, -0.00157565, 0.00916281, -0.02057706,
        0.02635537, -0.01647633, 0.00392377)
_I1S = (0.5, 0.87890594, 0.51498869, 0.15084934, 0.02658733, 0.00301532, 0.00032411)
_I1L = (0.39894228, -0.03988024, -0.00362018, 0.00163801, -0.01031555, 0.02282967,
        -0.02895312, 0.01787654, -0.00420059)


def _horner(c, u):
    v = 0.0
    for k in c[::-1]:
        v = v * u + k
    return v


def bessel_i0(x):
    """special.py:175-182."""
    if x <= 3.75:
        return _horner(_I0S, (x / 3.75) ** 2)
    return math.exp(x) / math.sqrt(x) * _horner(_I0L, 3.75 / x)


def bessel_i1(x):
    """special.py:185-192."""
    if x <= 3.75:
        return x * _horner(_I1S, (x / 3.75) ** 2)
    return math.exp(x) / math.sqrt(x) * _horner(_I1L, 3.75 / x)


def log_bessel_i0(x):
    """special.py:195-202."""
    if x <= 3.75:
        return math.log(_horner(_I0S, (x / 3.75) ** 2))
    return x - 0.5 * math.log(x) + math.log(_horner(_I0L, 3.75 / x))


def i1_i0_ratio(k):
    """special.py:205-217."""
    if k == 0.0:
        return 0.0
    if k <= 3.75:
        return bessel_i1(k) / bessel_i0(k)
    return _horner(_I1L, 3.75 / k) / _horner(_I0L, 3.75 / k)


# ----------------------------------------------------------------------------
# emission families: (family, params) tuples
#   ("gaussian", mu, sigma)   ("student_t", mu, sigma, nu)  ("gamma", shape, rate)
#   ("von_mises", mu, kappa)  ("poisson", rate)             ("joint", fam0, fam1)
# ----------------------------------------------------------------------------


def log_density(fam, y: np.ndarray, dtype=np.float64) -> np.ndarray:
    """Per-family _log_density in the reference's ufunc order.
    gaussian distributions.py:199-201, student_t :526-534, gamma :378-386,
    von_mises :359-360, poisson :256-260 (lgamma via math.lgamma, :80-86)."""
    R = dtype
    y = np.asarray(y, dtype=R)
    kind = fam[0]
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        if kind == "gaussian":
            mu, sigma = fam[1], fam[2]
            c0 = -0.5 * LOG_2PI - math.log(sigma)
            z = (y - R(mu)) / R(sigma)
            return R(c0) - (R(0.5) * z) * z
        if kind == "student_t":
            mu, sigma, nu = fam[1], fam[2], fam[3]
            c0 = (math.lgamma((nu + 1.0) / 2.0) - math.lgamma(nu / 2.0)
                  - 0.5 * math.log(nu * math.pi) - math.log(sigma))
            z = (y - R(mu)) / R(sigma)
            return R(c0) - R((nu + 1.0) / 2.0) * np.log1p((z * z) / R(nu))
        if kind == "gamma":
            shape, rate = fam[1], fam[2]
            c0 = shape * math.log(rate) - math.lgamma(shape)
            ly = np.log(np.where(y > 0, y, R(1.0)))
            d = (R(c0) + R(shape - 1.0) * ly) - R(rate) * y
            return np.where(y > 0, d, R(-np.inf)).astype(R)
        if kind == "von_mises":
            mu, kappa = fam[1], fam[2]
            return (R(kappa) * np.cos(y - R(mu)) - R(LOG_2PI)) - R(log_bessel_i0(kappa))
        if kind == "poisson":
            rate = fam[1]
            ok = (y >= 0) & (np.floor(y) == y)
            safe = np.where(ok, y, R(0.0))
            lg = np.array([math.lgamma(float(v) + 1.0) for v in safe], dtype=np.float64).astype(R)
            m = (safe * R(math.log(rate)) - R(rate)) - lg
            return np.where(ok, m, R(-np.inf)).astype(R)
    raise ValueError(kind)


def emission_matrix(emissions, obs, dtype=np.float64) -> np.ndarray:
    """inference.py:122-126 (column_stack of per-state log_prob); joint
    emissions add stream 0 then stream 1 (config-4 driver)."""
    cols = []
    for fam in emissions:
        if fam[0] == "joint":
            cols.append(log_density(fam[1], obs[:, 0], dtype) + log_density(fam[2], obs[:, 1], dtype))
        else:
            cols.append(log_density(fam, obs, dtype))
    return np.column_stack(cols).astype(dtype)


# ----------------------------------------------------------------------------
# recursions (inference.py)
# ----------------------------------------------------------------------------


def forward(log_pi, log_a, log_b):
    """inference.py:129-137."""
    T, K = log_b.shape
    la = np.empty((T, K))
    la[0] = log_pi + log_b[0]
    for t in range(1, T):
        la[t] = lse_axis(la[t - 1][:, None] + log_a, axis=0) + log_b[t]
    return la, float(lse_axis(la[-1][None, :], axis=1)[0])


def backward(log_a, log_b):
    """inference.py:140-146."""
    T, K = log_b.shape
    lb = np.zeros((T, K))
    for t in range(T - 2, -1, -1):
        lb[t] = lse_axis(log_a + (log_b[t + 1] + lb[t + 1])[None, :], axis=1)
    return lb


def posteriors(log_pi, log_a, log_b, include_xi=False):
    """inference.py:161-188 (returns dict; ll == -inf raises like the reference)."""
    la, ll = forward(log_pi, log_a, log_b)
    if ll == -np.inf:
        raise ValueError("sequence impossible under model")
    lb = backward(log_a, log_b)
    g = np.exp(la + lb - ll)
    xi = None
    if include_xi:
        T = log_b.shape[0]
        xi = np.stack([np.exp(la[t][:, None] + log_a + (log_b[t + 1] + lb[t + 1])[None, :] - ll)
                       for t in range(T - 1)]) if T > 1 else np.empty((0,) + log_a.shape)
    return {"log_alpha": la, "log_beta": lb, "ll": ll, "gamma": g, "xi": xi}


def viterbi(log_pi, log_a, log_b, dtype=np.float64):
    """inference.py:191-210, also returning the backpointer table (which the
    reference keeps local).  dtype=float32 restates it in float32."""
    R = dtype
    log_pi = np.asarray(log_pi, dtype=R)
    log_a = np.asarray(log_a, dtype=R)
    log_b = np.asarray(log_b, dtype=R)
    T, K = log_b.shape
    score = log_pi + log_b[0]
    back = np.zeros((T, K), dtype=np.int64)
    cols = np.arange(K)
    for t in range(1, T):
        cand = score[:, None] + log_a
        back[t] = np.argmax(cand, axis=0)
        score = cand[back[t], cols] + log_b[t]
    best = int(np.argmax(score))
    lj = float(score[best])
    path = np.empty(T, dtype=np.int64)
    path[-1] = best
    for t in range(T - 1, 0, -1):
        path[t - 1] = back[t, path[t]]
    return path, lj, back


# ----------------------------------------------------------------------------
# weighted fits (distributions.py) on (y, w) pairs restricted to w > 0
# ----------------------------------------------------------------------------


def _mv(y, w):
    """distributions.py:616-620 (two-pass)."""
    n = float(w.sum())
    m = float(np.dot(w, y) / n)
    return n, m, float(np.dot(w, (y - m) ** 2) / n)


def newton_1d(score, slope, x0, tol, max_iter=50):
    """distributions.py:732-761 (bracketed, safeguarded)."""
    lo, hi, x = 0.0, math.inf, x0
    for _ in range(max_iter):
        s = score(x)
        if abs(s) <= tol:
            return x, True
        if s > 0.0:
            lo = max(lo, x)
        else:
            hi = min(hi, x)
        d = slope(x)
        p = x - s / d if d != 0.0 else math.inf
        if not (math.isfinite(p) and lo < p < hi):
            p = x * 8.0 if math.isinf(hi) else 0.5 * (lo + hi)
        x = p
    return x, abs(score(x)) <= tol


def st_ll(y, w, mu, sigma, nu):
    """distributions.py:980-992."""
    z = (y - mu) / sigma
    per = (math.lgamma((nu + 1.0) / 2.0) - math.lgamma(nu / 2.0) - 0.5 * math.log(nu * math.pi)
           - math.log(sigma) - (nu + 1.0) / 2.0 * np.log1p(z * z / nu))
    return float(np.dot(w, per))


def fit(fam, y_all, w_all, ecme=(1e6, 1e-6, 50)):
    """refit (distributions.py:1094-1111) for the five hot-path families.
    Returns the new family tuple; raises ValueError with the reference text."""
    n_tot = float(w_all.sum())
    if n_tot <= 0.0:
        raise ValueError("fit requires positive total weight")
    keep = w_all > 0.0
    y, w = y_all[keep], w_all[keep]
    kind = fam[0]
    if kind == "gaussian":  # :632-636
        _, m, v = _mv(y, w)
        return ("gaussian", m, max(math.sqrt(v), SCALE_FLOOR))
    if kind == "poisson":  # :658-663
        if ((y < 0) | (np.floor(y) != y)).any():
            raise ValueError("poisson fit requires non-negative integer observations")
        _, m, _ = _mv(y, w)
        return ("poisson", max(m, SCALE_FLOOR))
    if kind == "gamma":  # :764-786
        if (y <= 0).any():
            raise ValueError("gamma fit requires strictly positive observations")
        n, m, v = _mv(y, w)
        if v <= 0.0:
            raise ValueError("gamma fit is degenerate: weighted variance is zero")
        c = math.log(m) - float(np.dot(w, np.log(y))) / n
        if c <= 0.0:
            raise ValueError("gamma fit is degenerate: zero log-moment gap")
        seed = m * m / v
        a, ok = newton_1d(lambda x: math.log(x) - digamma(x) - c,
                          lambda x: 1.0 / x - trigamma(x), seed, 1e-10)
        if not ok:
            warnings.warn("gamma shape update did not converge; using moment seed", RuntimeWarning)
            a = seed
        return ("gamma", a, a / m)
    if kind == "von_mises":  # :874-916
        n = n_tot
        if not np.isfinite(y).all():
            raise ValueError("von_mises fit requires finite angles")
        s, c = float(np.dot(w, np.sin(y))), float(np.dot(w, np.cos(y)))
        mu = math.atan2(s, c)
        if mu <= -math.pi:
            mu = math.pi
        rbar = math.hypot(s, c) / n
        if rbar <= 1e-12:
            return ("von_mises", mu, 0.0)
        if rbar >= 1.0 - 1e-12:
            return ("von_mises", mu, KAPPA_CEIL)
        k = rbar * (2.0 - rbar * rbar) / (1.0 - rbar * rbar)
        for _ in range(50):
            A = i1_i0_ratio(k)
            f = A - rbar
            if abs(f) <= 1e-10:
                break
            step = f / (1.0 - A * A - A / k)
            p = k - step
            while p <= 0.0:
                step *= 0.5
                p = k - step
            k = p
            if k >= KAPPA_CEIL:
                k = KAPPA_CEIL
                break
        return ("von_mises", mu, k)
    if kind == "student_t":  # :1031-1087 (one ECME cycle)
        mu, sig, nu, _ = student_t_cycle(y, w, n_tot, fam[1], fam[2], fam[3], ecme)
        return ("student_t", mu, sig, nu)
    raise ValueError(kind)


def student_t_cycle(y, w, n_tot, mu0, s0, nu0, ecme=(1e6, 1e-6, 50)):
    """One ECME cycle (distributions.py:1031-1087) on the w>0 entries; also
    returns how many guard halvings the likelihood guard took (0 = the Newton
    proposal passed, 60 = fell back to nu0)."""
    if True:
        nu_ceil, nu_tol, max_newton = ecme
        n = n_tot
        u = (nu0 + 1.0) / (nu0 + ((y - mu0) / s0) ** 2)
        wu = w * u
        mu = float(np.dot(wu, y) / wu.sum())
        sig = max(math.sqrt(float(np.dot(wu, (y - mu) ** 2) / n)), SCALE_FLOOR)
        half = (nu0 + 1.0) / 2.0
        mix = float(np.dot(w, np.log(u) - u)) + n * (digamma(half) - math.log(half))

        def q(v):
            return n * (v / 2.0 * math.log(v / 2.0) - math.lgamma(v / 2.0)) + v / 2.0 * mix

        nu = nu0
        for _ in range(max_newton):
            sc = n / 2.0 * (math.log(nu / 2.0) + 1.0 - digamma(nu / 2.0)) + mix / 2.0
            h = n / 4.0 * (2.0 / nu - trigamma(nu / 2.0))
            step = -sc / h
            p = nu + step
            while p <= 0.0:
                step *= 0.5
                p = nu + step
            qn = q(nu)
            while q(p) < qn and abs(step) > 1e-300:
                step *= 0.5
                p = nu + step
            if p >= nu_ceil:
                nu = nu_ceil
                break
            moved = abs(p - nu)
            nu = p
            if moved < nu_tol:
                break
        base = st_ll(y, w, mu, sig, nu0)
        halvings = 60
        for k in range(60):
            if st_ll(y, w, mu, sig, nu) >= base - 1e-12:
                halvings = k
                break
            nu = nu0 + 0.5 * (nu - nu0)
        else:
            nu = nu0
        return mu, sig, nu, halvings


# ----------------------------------------------------------------------------
# exhaustive path enumeration (the reference's tests/oracles.py:281-350 used by
# test_acceptance.py:70-91 and test_inference.py): tiny K, T only
# ----------------------------------------------------------------------------


def enumerate_paths(log_pi, log_a, log_b):
    """Joint log-probability of every state path, lexicographic order."""
    import itertools

    T, K = log_b.shape
    out = []
    for path in itertools.product(range(K), repeat=T):
        lp = log_pi[path[0]] + log_b[0, path[0]]
        for t in range(1, T):
            lp += log_a[path[t - 1], path[t]] + log_b[t, path[t]]
        out.append((path, float(lp)))
    return out


def brute_force(log_pi, log_a, log_b):
    """(log-likelihood, gamma [T, K], best path, best joint) by enumeration;
    the best path is the first (lexicographically smallest) maximiser."""
    paths = enumerate_paths(log_pi, log_a, log_b)
    lps = np.array([lp for _, lp in paths])
    mx = lps.max()
    ll = float(mx + math.log(np.exp(lps - mx).sum())) if np.isfinite(mx) else -math.inf
    T, K = log_b.shape
    g = np.zeros((T, K))
    for (path, lp) in paths:
        if np.isfinite(lp):
            w = math.exp(lp - ll)
            for t, s in enumerate(path):
                g[t, s] += w
    best = int(np.argmax(lps))
    return ll, g, tuple(paths[best][0]), float(lps[best])


# ----------------------------------------------------------------------------
# Baum-Welch (training.py:160-236) over a list of sequences
# ----------------------------------------------------------------------------


def model_tables(pi, A):
    with np.errstate(divide="ignore"):
        return np.log(np.asarray(pi, float)), np.log(np.asarray(A, float))


def estep_sequence(args):
    """One sequence of training.py:188-210; returns its contributions.
    Top-level so it can run in a multiprocessing pool."""
    s_idx, y, pi, A, emissions = args
    log_pi, log_a = model_tables(pi, A)
    lb = emission_matrix(emissions, y)
    dead = np.nonzero(~(lb > -np.inf).any(axis=1))[0]
    if dead.size:
        return {"error": ("dead", s_idx, int(dead[0]))}
    la, ll = forward(log_pi, log_a, lb)
    if ll == -np.inf:
        return {"error": ("impossible", s_idx)}
    lbeta = backward(log_a, lb)
    g = np.exp(la + lbeta - ll)
    K = len(pi)
    xi = np.zeros((K, K))
    for t in range(len(y) - 1):
        xi += np.exp(la[t][:, None] + log_a + (lb[t + 1] + lbeta[t + 1])[None, :] - ll)
    return {"ll": ll, "g0": g[0], "gamma": g, "gtot": g[:-1].sum(axis=0), "xi": xi}


def baum_welch(pi, A, emissions, seqs, max_iterations, rel_tol=1e-300, eps=1e-8, pool=None):
    """training.py:160-236 with emissions as family tuples.  Returns
    (pi, A, emissions, trace, converged, collapsed)."""
    pi = np.asarray(pi, float)
    A = np.asarray(A, float)
    emissions = list(emissions)
    K = len(pi)
    seqs = [np.asarray(s, float) for s in seqs]
    all_obs = np.concatenate(seqs, axis=0)
    trace, collapsed, converged = [], [], False
    for it in range(1, max_iterations + 1):
        jobs = [(i, s, pi, A, emissions) for i, s in enumerate(seqs)]
        res = pool.map(estep_sequence, jobs) if pool is not None else [estep_sequence(j) for j in jobs]
        total = 0.0
        xi = np.zeros((K, K))
        gtot = np.zeros(K)
        for r in res:
            if "error" in r:
                e = r["error"]
                if e[0] == "dead":
                    raise ValueError(f"observation outside the support of every state: sequence {e[1]}, index {e[2]}")
                raise ValueError(f"sequence {e[1]} is impossible under the model")
            total += r["ll"]
            xi += r["xi"]
            gtot += r["gtot"]
        trace.append(total)
        if len(trace) >= 2:
            d = trace[-1] - trace[-2]
            if d == 0.0 or abs(d) < rel_tol * abs(trace[-1]):
                converged = True
                break
        if it == max_iterations:
            break
        G = np.concatenate([r["gamma"] for r in res], axis=0)
        new_em = []
        for j, fam in enumerate(emissions):
            w = G[:, j]
            if float(w.sum()) < eps:
                new_em.append(fam)
                collapsed.append((it, j))
                continue
            if fam[0] == "joint":
                new_em.append(("joint", fit(fam[1], all_obs[:, 0], w), fit(fam[2], all_obs[:, 1], w)))
            else:
                new_em.append(fit(fam, all_obs, w))
        # training.py:105-127
        newpi = np.mean(np.stack([r["g0"] for r in res]), axis=0)
        newpi = newpi / newpi.sum()
        newA = np.array(A, copy=True)
        for i in range(K):
            if gtot[i] >= eps:
                row = xi[i] / gtot[i]
                tot = row.sum()
                if tot > 0:
                    newA[i] = row / tot
        pi, A, emissions = newpi, newA, new_em
    return pi, A, emissions, trace, converged, collapsed
