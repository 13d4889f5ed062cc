"""GPU parity of the training path: the benched pipeline step, fp32
Baum-Welch, the reference's forced M-step paths and the reference's own
training / acceptance tests, against the CPU oracle.

Tolerances (BASELINE.json north_star, plus the fp32 parameter bound stated in
DESIGN.md §4):
  fp64: LL, statistics totals and updated parameters <= 1e-9 relative
        (probabilities <= 1e-9 absolute)
  fp32: LL <= 1e-4 relative, posteriors <= 1e-5 absolute; statistics totals
        and updated parameters <= 1e-4 relative (probabilities <= 1e-5
        absolute) -- the fp32 posteriors' 1e-5 bound summed into weighted
        totals
"""

import math
import warnings

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import loghmm_oracle as O  # noqa: E402

import paper_2605_29208_b200 as H  # noqa: E402
from paper_2605_29208_b200 import engine  # noqa: E402
from paper_2605_29208_b200.configs import make_config  # noqa: E402
from paper_2605_29208_b200.pipeline import Pipeline  # noqa: E402

from test_gpu_parity import to_model, to_tuples  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


TOL = {"float64": dict(ll=1e-9, tot=1e-9, par=1e-9, prob=1e-9),
       "float32": dict(ll=1e-4, tot=1e-4, par=1e-4, prob=1e-5)}


def _r32(data, dtype):
    """The observations the kernel sees (fp32 inputs are rounded first)."""
    return data.astype(np.float32).astype(np.float64) if dtype == "float32" else data


def _oracle_totals(model, seqs):
    """xi totals, gamma totals (t < T-1), sum of first gammas and total LL
    (training.py:180-210) from the oracle's per-sequence E-step."""
    K = model.num_states
    xi, gt, g0, ll = np.zeros((K, K)), np.zeros(K), np.zeros(K), 0.0
    for i, y in enumerate(seqs):
        r = O.estep_sequence((i, y, model.initial, model.transitions, to_tuples(model)))
        xi += r["xi"]
        gt += r["gtot"]
        g0 += r["g0"]
        ll += r["ll"]
    return xi, gt, g0, ll


def _check_params(fitted_tuples, oracle_tuples, tol):
    for a, b in zip(fitted_tuples, oracle_tuples):
        assert a[0] == b[0]
        if a[0] == "joint":
            np.testing.assert_allclose(a[1][1:], b[1][1:], rtol=tol)
            np.testing.assert_allclose(a[2][1:], b[2][1:], rtol=tol)
        else:
            np.testing.assert_allclose(a[1:], b[1:], rtol=tol)


# ---------------------------------------------------------------------------
# the benched step (Pipeline: fused reduction + M-step) against the oracle
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,B,T", [("c2", 64, 1024), ("c3", 16, 2048), ("c4", 16, 2000)])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_pipeline_step_matches_oracle(name, B, T, dtype):
    """Pipeline.run() -- FB || Viterbi, the fused reduce_mstep kernel, the
    variance pass and the full ECME guard -- gives the oracle's statistics
    totals, total LL and one-M-step model (O.baum_welch, 2 iterations)."""
    if name == "c3" and dtype == "float32":
        pytest.skip("c3 is fp64 in BASELINE.json")
    cfg = make_config(name, B=B, T=T)
    tol = TOL[dtype]
    p = Pipeline(cfg.init, B, T, dtype)
    td = torch.float32 if dtype == "float32" else torch.float64
    p.load(torch.from_numpy(cfg.data).to(td))
    p.run()
    torch.cuda.synchronize()
    collapsed = p.check()
    assert collapsed == []
    seqs = [_r32(cfg.data[b], dtype) for b in range(B)]
    xi, gt, g0, ll = _oracle_totals(cfg.init, seqs)
    K = cfg.K
    tot = p.totals.cpu().numpy()
    np.testing.assert_allclose(tot[: K * K].reshape(K, K), xi, rtol=tol["tot"])
    np.testing.assert_allclose(tot[K * K: K * K + K], gt, rtol=tol["tot"])
    np.testing.assert_allclose(tot[K * K + K: K * K + 2 * K], g0, rtol=tol["tot"], atol=tol["prob"] * B)
    assert tot[-1] == pytest.approx(ll, rel=tol["ll"])
    pi, A, em, trace, _, _ = O.baum_welch(cfg.init.initial, cfg.init.transitions, to_tuples(cfg.init),
                                          seqs, 2)
    upd = p.updated_model()
    np.testing.assert_allclose(upd.transitions, A, atol=tol["prob"])
    np.testing.assert_allclose(upd.initial, pi, atol=tol["prob"])
    _check_params(to_tuples(upd), em, tol["par"])
    # the Viterbi leg of the same step
    lp, la = O.model_tables(cfg.init.initial, cfg.init.transitions)
    for b in (0, B - 1):
        if dtype == "float64":
            path, lj, _ = O.viterbi(lp, la, O.emission_matrix(to_tuples(cfg.init), cfg.data[b]))
        else:
            path, lj, _ = O.viterbi(lp.astype(np.float32), la.astype(np.float32),
                                    O.emission_matrix(to_tuples(cfg.init), cfg.data[b].astype(np.float32),
                                                      np.float32), np.float32)
        if name in ("c2",):  # IEEE-basic-op family: bit-exact
            assert np.array_equal(p.vit.path[b * T:(b + 1) * T].cpu().numpy(), path)
            assert p.vit.log_joint[b].item() == lj


@pytest.mark.parametrize("name,B,T,iters", [("c2", 32, 1024, 3), ("c3", 8, 2048, 3), ("c4", 8, 2000, 3)])
def test_baum_welch_fp32_matches_oracle(name, B, T, iters):
    """fp32 training (the fp32 chunk-operator kernel's statistics + the
    M-step) against the fp64 oracle on the fp32-rounded observations."""
    cfg = make_config(name, B=B, T=T)
    data = [_r32(cfg.data[b], "float32") for b in range(B)]
    fitted, rep = H.baum_welch(cfg.init, [cfg.data[b] for b in range(B)],
                               H.TrainingConfig(max_iterations=iters, rel_tol=1e-300), dtype="float32")
    pi, A, em, trace, _, _ = O.baum_welch(cfg.init.initial, cfg.init.transitions, to_tuples(cfg.init),
                                          data, iters)
    tol = TOL["float32"]
    np.testing.assert_allclose(rep.log_likelihood_trace, trace, rtol=tol["ll"])
    np.testing.assert_allclose(fitted.transitions, A, atol=tol["prob"])
    np.testing.assert_allclose(fitted.initial, pi, atol=tol["prob"])
    _check_params(to_tuples(fitted), em, tol["par"])


# ---------------------------------------------------------------------------
# forced M-step paths
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_variance_second_pass_forced(dtype):
    """A state initialised 100 sigma away from its data: the shifted one-pass
    variance would cancel catastrophically, so the M-step flags the state and
    the exact two-pass variance (distributions.py:616-620) runs."""
    rng = np.random.default_rng(21)
    seqs = [np.concatenate([rng.normal(0.0, 1.0, 300), rng.normal(50.0, 2.0, 300)]) for _ in range(4)]
    m = H.HmmModel([0.5, 0.5], [[0.95, 0.05], [0.05, 0.95]], (H.Gaussian(100.0, 1.0), H.Gaussian(-60.0, 1.0)))
    fitted, rep = H.baum_welch(m, seqs, H.TrainingConfig(max_iterations=3, rel_tol=1e-300), dtype=dtype)
    data = [_r32(s, dtype) for s in seqs]
    pi, A, em, trace, _, _ = O.baum_welch(m.initial, m.transitions, to_tuples(m), data, 3)
    tol = TOL[dtype]
    np.testing.assert_allclose(rep.log_likelihood_trace, trace, rtol=tol["ll"])
    _check_params(to_tuples(fitted), em, tol["par"])
    # and through the pipeline (fixed-shape step)
    p = Pipeline(m, 4, 600, dtype)
    p.load(torch.from_numpy(np.stack(seqs)))
    p.run()
    torch.cuda.synchronize()
    p.check()
    pi1, A1, em1, _, _, _ = O.baum_welch(m.initial, m.transitions, to_tuples(m), data, 2)
    _check_params(to_tuples(p.updated_model()), em1, tol["par"])


def test_workspace_counter_survives_shape_changes():
    """a larger-K Student-t fit followed by a smaller-K fit
    whose variance pass is flagged, in one process (shared workspaces): the
    second fit still finishes its flagged states exactly."""
    rng = np.random.default_rng(5)
    K = 8
    big = H.HmmModel(np.full(K, 1 / K), np.full((K, K), 1 / K),
                     tuple(H.StudentT(float(k), 1.0, 5.0) for k in range(K)))
    ys = [rng.standard_t(4.0, 40_000) + rng.integers(0, K, 40_000) for _ in range(3)]
    H.baum_welch(big, ys, H.TrainingConfig(max_iterations=2, rel_tol=1e-300))
    seqs = [np.concatenate([rng.normal(0.0, 1.0, 300), rng.normal(50.0, 2.0, 300)]) for _ in range(4)]
    m = H.HmmModel([0.5, 0.5], [[0.95, 0.05], [0.05, 0.95]], (H.Gaussian(100.0, 1.0), H.Gaussian(-60.0, 1.0)))
    fitted, rep = H.baum_welch(m, seqs, H.TrainingConfig(max_iterations=3, rel_tol=1e-300))
    pi, A, em, trace, _, _ = O.baum_welch(m.initial, m.transitions, to_tuples(m), seqs, 3)
    _check_params(to_tuples(fitted), em, 1e-9)


def _guard_case(min_halvings=9):
    """A K=1 Student-t problem whose ECME likelihood guard needs more halvings
    than one candidate batch holds (found by a seeded search; the oracle
    counts the halvings)."""
    rng = np.random.default_rng(1)
    for _ in range(2000):
        n = int(rng.integers(50, 300))
        y = rng.standard_t(rng.uniform(0.5, 30), n) * rng.uniform(0.1, 3)
        mu0, s0, nu0 = rng.normal(0, 1), rng.uniform(0.05, 3), float(np.exp(rng.uniform(-1, 5)))
        k = O.student_t_cycle(y, np.ones(n), float(n), mu0, s0, nu0)[3]
        if min_halvings <= k < 60:
            return y, float(mu0), float(s0), nu0, k
    raise AssertionError("no guard case found")


def test_student_t_guard_many_candidates():
    """The guard walks past the first candidate batches (training polls
    need_more; the pipeline launches the fixed batches) and lands on the
    reference's candidate."""
    y, mu0, s0, nu0, k = _guard_case()
    m = H.HmmModel([1.0], [[1.0]], (H.StudentT(mu0, s0, nu0),))
    fitted, rep = H.baum_welch(m, [y], H.TrainingConfig(max_iterations=2, rel_tol=1e-300))
    pi, A, em, trace, _, _ = O.baum_welch([1.0], [[1.0]], to_tuples(m), [y], 2)
    np.testing.assert_allclose(rep.log_likelihood_trace, trace, rtol=1e-9)
    _check_params(to_tuples(fitted), em, 1e-9)
    p = Pipeline(m, 1, len(y), "float64")
    p.load(torch.from_numpy(y[None]))
    p.run()
    torch.cuda.synchronize()
    p.check()
    _check_params(to_tuples(p.updated_model()), em, 1e-9)
    assert int(p.status.cpu()[0]) & H._native.MS_STUDENT_GUARD == 0


def test_gamma_constant_data_error_names_state():
    """test_training.py:129-138: the fit error carries the state index."""
    m = H.HmmModel([1.0], [[1.0]], (H.Gamma(1.0, 1.0),))
    with pytest.raises(H.TrainingError, match="state 0: gamma fit is degenerate: weighted variance is zero"):
        H.baum_welch(m, [np.array([1.0, 1.0])], H.TrainingConfig(max_iterations=2))
    p = Pipeline(m, 1, 2, "float64")
    p.load(torch.tensor([[1.0, 1.0]], dtype=torch.float64))
    p.run()
    torch.cuda.synchronize()
    with pytest.raises(H.TrainingError, match="state 0: gamma fit is degenerate"):
        p.check()


def test_fit_warnings_surface():
    """FitWarning paths (distributions.py:890-893, :1070): a von Mises state on
    constant angles clamps at the boundary; a Student-t state on Gaussian
    data clamps its degrees of freedom."""
    m = H.HmmModel([1.0], [[1.0]], (H.VonMises(0.5, 1.0),))
    with pytest.warns(H.FitWarning, match="resultant length is at the boundary"):
        fitted, _ = H.baum_welch(m, [np.full(50, 0.25)], H.TrainingConfig(max_iterations=2))
    assert fitted.emissions[0].kappa == 1e5
    rng = np.random.default_rng(3)
    y = rng.normal(0.0, 1.0, 20_000)
    m2 = H.HmmModel([1.0], [[1.0]], (H.StudentT(0.0, 1.0, 1e5),))
    pi, A, em, trace, _, _ = O.baum_welch([1.0], [[1.0]], to_tuples(m2), [y], 2)
    if em[0][3] == 1e6:  # the oracle clamps too: the warning must surface
        with pytest.warns(H.FitWarning, match="degrees of freedom clamped"):
            fitted2, _ = H.baum_welch(m2, [y], H.TrainingConfig(max_iterations=2, rel_tol=1e-300))
    else:
        fitted2, _ = H.baum_welch(m2, [y], H.TrainingConfig(max_iterations=2, rel_tol=1e-300))
    _check_params(to_tuples(fitted2), em, 1e-9)


# ---------------------------------------------------------------------------
# ports of the reference's own tests
# ---------------------------------------------------------------------------
def test_collapse_guard_unreachable_state_frozen():
    """test_training.py:158-175 and test_acceptance.py:336-362 (end to end):
    an unreachable state keeps its distribution object, every M-step records
    it as collapsed, the trace never dips."""
    for frozen, seed, n, iters in ((H.Gaussian(42.0, 7.0), 5, 60, 10), (H.StudentT(1.25, 2.5, 7.5), 5, 80, 12)):
        model = H.HmmModel([1.0, 0.0], [[1.0, 0.0], [0.0, 1.0]], (H.Gaussian(0.0, 1.0), frozen))
        seq = np.random.default_rng(seed).normal(size=n)
        fitted, report = H.baum_welch(model, [seq], H.TrainingConfig(max_iterations=iters))
        assert fitted.emissions[1] is frozen
        assert report.collapsed_states
        assert all(state == 1 for _, state in report.collapsed_states)
        trace = report.log_likelihood_trace
        assert all(b >= a - 1e-7 for a, b in zip(trace, trace[1:]))
        pi, A, em, otrace, _, ocol = O.baum_welch(model.initial, model.transitions, to_tuples(model), [seq],
                                                  iters, rel_tol=1e-8)
        np.testing.assert_allclose(trace, otrace, rtol=1e-9)
        assert [tuple(c) for c in report.collapsed_states] == [tuple(c) for c in ocol]


def test_label_permutation_equivariance_two_states():
    """test_training.py:177-197: exact (abs=0) trace equality and bit-equal
    parameters under a label swap."""
    rng = np.random.default_rng(6)
    seq = np.concatenate([rng.normal(0, 1, 40), rng.normal(4, 1, 40)])
    base = H.HmmModel([0.7, 0.3], [[0.8, 0.2], [0.3, 0.7]], (H.Gaussian(0.5, 1.2), H.Gaussian(3.5, 0.9)))
    swapped = H.HmmModel([0.3, 0.7], [[0.7, 0.3], [0.2, 0.8]], (H.Gaussian(3.5, 0.9), H.Gaussian(0.5, 1.2)))
    cfg = H.TrainingConfig(max_iterations=25)
    m1, r1 = H.baum_welch(base, [seq], cfg)
    m2, r2 = H.baum_welch(swapped, [seq], cfg)
    assert r1.log_likelihood_trace == pytest.approx(r2.log_likelihood_trace, abs=0)
    assert m1.initial.tolist() == m2.initial[::-1].tolist()
    assert np.array_equal(m1.transitions, m2.transitions[::-1, ::-1])
    assert m1.emissions == (m2.emissions[1], m2.emissions[0])


def test_label_permutation_equivariance_three_states():
    """test_training.py:199-219."""
    rng = np.random.default_rng(7)
    seq = np.concatenate([rng.normal(0, 1, 30), rng.normal(5, 1, 30), rng.normal(10, 1, 30)])
    perm = [2, 0, 1]
    pi = np.array([0.5, 0.3, 0.2])
    a = np.array([[0.8, 0.1, 0.1], [0.2, 0.6, 0.2], [0.1, 0.3, 0.6]])
    em = (H.Gaussian(0.5, 1.0), H.Gaussian(4.5, 1.0), H.Gaussian(9.5, 1.0))
    base = H.HmmModel(pi, a, em)
    inv = np.argsort(perm)
    permuted = H.HmmModel(pi[perm], a[np.ix_(perm, perm)], tuple(em[i] for i in perm))
    cfg = H.TrainingConfig(max_iterations=8)
    m1, r1 = H.baum_welch(base, [seq], cfg)
    m2, r2 = H.baum_welch(permuted, [seq], cfg)
    assert r1.log_likelihood_trace == pytest.approx(r2.log_likelihood_trace, abs=1e-8)
    assert np.allclose(m1.initial, m2.initial[inv], atol=1e-9)
    assert np.allclose(m1.transitions, m2.transitions[np.ix_(inv, inv)], atol=1e-9)
    for i in range(3):
        assert m1.emissions[i].mu == pytest.approx(m2.emissions[inv[i]].mu, abs=1e-9)


def test_brute_force_inference_equivalence():
    """test_acceptance.py:70-91, Gaussian models (K in {2,3}, T in {4..8}):
    LL and gamma within 1e-10 of exhaustive enumeration, Viterbi path exact,
    log joint within 1e-10."""
    rng = np.random.default_rng(2024)
    checked = 0
    for i in range(200):
        k = 2 + (i % 2)
        t_len = 4 + (i % 5)
        pi = rng.dirichlet(np.ones(k))
        a = rng.dirichlet(np.ones(k), size=k)
        m = H.HmmModel(pi, a, tuple(H.Gaussian(float(rng.normal(0, 2)), float(rng.uniform(0.3, 2.0)))
                                    for _ in range(k)))
        seq = rng.normal(size=t_len) * 2.0
        lp, la = O.model_tables(pi, a)
        ll, g, path, joint = O.brute_force(lp, la, O.emission_matrix(to_tuples(m), seq))
        fb = H.posteriors(m, seq)
        assert fb.log_likelihood == pytest.approx(ll, abs=1e-10)
        assert np.allclose(fb.gamma, g, atol=1e-10)
        vit = H.viterbi(m, seq)
        assert tuple(vit.path) == path
        assert vit.log_joint == pytest.approx(joint, abs=1e-10)
        checked += 1
    assert checked == 200


def test_multi_sequence_total_and_empty_data():
    """test_training.py:222-241: the trace's last entry is the sum of the
    per-sequence LLs; empty data is a TrainingError."""
    rng = np.random.default_rng(8)
    s1, s2 = rng.normal(0, 1, 30), rng.normal(2, 1, 45)
    model = H.default_initial_model(2, "gaussian", [s1, s2])
    fitted, report = H.baum_welch(model, [s1, s2], H.TrainingConfig(max_iterations=20))
    _, ll1 = H.forward_log(fitted, s1)
    _, ll2 = H.forward_log(fitted, s2)
    assert report.log_likelihood_trace[-1] == pytest.approx(ll1 + ll2, abs=1e-9)
    with pytest.raises(H.TrainingError):
        H.baum_welch(H.HmmModel([1.0], [[1.0]], (H.Gaussian(0, 1),)), [])


# ---------------------------------------------------------------------------
# NaN validation on every entry point
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("K", [3, 12])
def test_nan_rejected_everywhere(K):
    m = H.HmmModel(np.full(K, 1 / K), np.full((K, K), 1 / K),
                   tuple(H.Gaussian(float(k), 1.0) for k in range(K)))
    y = np.linspace(-1, 1, 64)
    y[17] = np.nan
    for fn in (lambda: H.viterbi(m, y), lambda: H.posteriors(m, y), lambda: H.emission_log_matrix(m, y),
               lambda: H.viterbi_batch(m, [y, y.copy()]), lambda: H.viterbi_batch(m, np.stack([y, y])),
               lambda: H.viterbi_batch(m, [y], dtype="float32")):
        with pytest.raises(ValueError, match="observation sequence contains NaN"):
            fn()


# ---------------------------------------------------------------------------
# the scaled recursions against an unreachable best-emission state
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("layout", ["equal", "ragged"])
def test_unreachable_best_emission_state(dtype, layout):
    """State 2 is unreachable (pi_2 = 0, column 2 of A is zero) and its
    emission beats the reachable states by ~100 nats at every step: the
    linear scaled recursions must follow the best ENTERABLE state
    (load_colscaled), so the sequence stays feasible with the reference's
    finite LL (fp32's range ends ~87 nats below the shift)."""
    rng = np.random.default_rng(11)
    A = np.array([[0.9, 0.1, 0.0], [0.2, 0.8, 0.0], [0.5, 0.5, 0.0]])
    m = H.HmmModel([0.6, 0.4, 0.0], A, (H.Gaussian(14.0, 1.0), H.Gaussian(14.5, 1.0), H.Gaussian(0.0, 1.0)))
    T = 64
    seqs = [rng.normal(0.0, 0.3, T) for _ in range(5)]
    if layout == "ragged":
        seqs = [s[: T - 7 * i] for i, s in enumerate(seqs)]
    r = H.posteriors_batch(m, seqs, dtype=dtype, include_xi=layout == "ragged")
    lp, la = O.model_tables(m.initial, m.transitions)
    tol = TOL[dtype]
    for b, y in enumerate(seqs):
        o = O.posteriors(lp, la, O.emission_matrix(to_tuples(m), _r32(y, dtype)))
        assert math.isfinite(o["ll"]) and o["ll"] < -90 * len(y)
        s = slice(r.offsets[b], r.offsets[b + 1])
        assert r.log_likelihood[b].item() == pytest.approx(o["ll"], rel=tol["ll"])
        np.testing.assert_allclose(r.gamma[s].double().cpu().numpy(), o["gamma"], atol=tol["prob"])
    fitted, rep = H.baum_welch(m, seqs, H.TrainingConfig(max_iterations=2, rel_tol=1e-300), dtype=dtype)
    pi, A2, em, trace, _, _ = O.baum_welch(m.initial, m.transitions, to_tuples(m),
                                           [_r32(s, dtype) for s in seqs], 2)
    np.testing.assert_allclose(rep.log_likelihood_trace, trace, rtol=tol["ll"])
    np.testing.assert_allclose(fitted.transitions, A2, atol=tol["prob"])
