"""The drop-in shim (paper_2605_29208_b200.compat) under the reference
package itself: the unmodified ``loghmm`` installed in baseline/_ref (the
bench's reference install; skipped where it is absent) is rebound to the B200
core, and checks restating the reference's own inference / training tests
(test_inference.py:79-280, test_training.py:114-175) run through the
reference's public API.  Expected values come from the same ``loghmm`` with
its original functions (saved before the install), so every comparison is
"reference on the CPU" vs "reference API on the GPU" on identical inputs.
"""

import itertools
import math
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not (REF / "loghmm").exists():
        pytest.skip("reference install baseline/_ref absent")
    sys.path.insert(0, str(REF))
    import loghmm

    from paper_2605_29208_b200 import compat

    import loghmm.inference
    import loghmm.training

    orig = {n: getattr(loghmm.inference, n) for n in ("posteriors", "viterbi", "forward_log",
                                                       "backward_log", "emission_log_matrix")}
    orig.update({n: getattr(loghmm.training, n) for n in ("baum_welch", "score_model")})
    handle = compat.install(loghmm)
    yield loghmm, orig
    handle.uninstall()


def rand_gauss(L, rng, k):
    pi = rng.dirichlet(np.ones(k))
    a = rng.dirichlet(np.ones(k), size=k)
    return L.HmmModel(pi, a, tuple(L.Gaussian(float(rng.normal(0, 2)), float(rng.uniform(0.3, 2.0)))
                                   for _ in range(k)))


def rand_cat(L, rng, k, m=3):
    pi = rng.dirichlet(np.ones(k))
    a = rng.dirichlet(np.ones(k), size=k)
    return L.HmmModel(pi, a, tuple(L.Categorical(tuple(rng.dirichlet(np.ones(m)))) for _ in range(k)))


def test_results_are_reference_types_and_values(L):
    loghmm, orig = L
    rng = np.random.default_rng(1)
    for make in (rand_gauss, rand_cat):
        m = make(loghmm, rng, 3)
        seq = rng.normal(size=40) * 2.0 if make is rand_gauss else rng.integers(0, 3, 40).astype(float)
        fb = loghmm.posteriors(m, seq, include_xi=True)
        ref = orig["posteriors"](m, seq, include_xi=True)
        assert type(fb) is loghmm.inference.ForwardBackwardResult
        assert fb.log_likelihood == pytest.approx(ref.log_likelihood, rel=1e-12)
        np.testing.assert_allclose(fb.gamma, ref.gamma, atol=1e-12)
        np.testing.assert_allclose(fb.xi, ref.xi, atol=1e-12)
        vt, vr = loghmm.viterbi(m, seq), orig["viterbi"](m, seq)
        assert type(vt) is loghmm.inference.ViterbiResult
        assert np.array_equal(vt.path, vr.path) and vt.log_joint == vr.log_joint


def test_forward_backward_identities(L):
    """test_inference.py TestForward / TestBackward through the shim."""
    loghmm, orig = L
    m1 = loghmm.HmmModel([1.0], [[1.0]], (loghmm.Gaussian(0.0, 1.0),))
    seq = [0.3, -1.2, 0.9]
    _, ll = loghmm.forward_log(m1, seq)
    assert ll == pytest.approx(sum(float(m1.emissions[0].log_prob(v)) for v in seq), abs=1e-12)
    rng = np.random.default_rng(0)
    m = rand_gauss(loghmm, rng, 3)
    la, ll = loghmm.forward_log(m, [0.4])
    exp0 = m.log_initial() + loghmm.inference.emission_log_matrix(m, [0.4])[0]
    assert np.allclose(la[0], exp0, atol=1e-13)
    m_u = loghmm.HmmModel([1.0], [[1.0]], (loghmm.Uniform(0.0, 1.0),))
    _, ll = loghmm.forward_log(m_u, [0.5, 4.0, 0.5])
    assert ll == -math.inf
    rng = np.random.default_rng(3)
    m = rand_gauss(loghmm, rng, 3)
    seq = rng.normal(size=9)
    la, ll = loghmm.forward_log(m, seq)
    lb = loghmm.backward_log(m, seq)
    assert (lb[-1] == 0.0).all()
    for t in range(len(seq)):
        v = la[t] + lb[t]
        mx = v.max()
        assert mx + math.log(np.exp(v - mx).sum()) == pytest.approx(ll, abs=1e-9)


def test_backward_matches_suffix_enumeration(L):
    loghmm, orig = L
    rng = np.random.default_rng(4)
    m = rand_cat(loghmm, rng, 2)
    seq = rng.integers(0, 3, size=5).astype(float)
    lbeta = loghmm.backward_log(m, seq)
    la, lbm = m.log_transitions(), orig["emission_log_matrix"](m, seq)
    T, K = len(seq), m.num_states
    for t in range(T):
        for i in range(K):
            terms = []
            for suffix in itertools.product(range(K), repeat=T - 1 - t):
                lp, prev = 0.0, i
                for step, st in enumerate(suffix):
                    lp += la[prev, st] + lbm[t + 1 + step, st]
                    prev = st
                terms.append(lp)
            if terms:
                mx = max(terms)
                exp = mx + math.log(sum(math.exp(x - mx) for x in terms))
            else:
                exp = 0.0
            assert lbeta[t, i] == pytest.approx(exp, abs=1e-10)


def test_posteriors_and_viterbi_contracts(L):
    """test_inference.py TestPosteriors / TestViterbi / TestStability."""
    loghmm, orig = L
    det = loghmm.HmmModel([1.0, 0.0], [[1.0, 0.0], [0.0, 1.0]],
                          (loghmm.Uniform(0.0, 1.0), loghmm.Uniform(10.0, 11.0)))
    fb = loghmm.posteriors(det, [0.5, 0.2, 0.9])
    assert np.allclose(fb.gamma, np.column_stack([np.ones(3), np.zeros(3)]))
    rng = np.random.default_rng(5)
    for _ in range(10):
        m = rand_gauss(loghmm, rng, 3)
        assert np.allclose(loghmm.posteriors(m, rng.normal(size=20)).gamma.sum(axis=1), 1.0, atol=1e-9)
    rng = np.random.default_rng(7)
    m = rand_gauss(loghmm, rng, 3)
    fb = loghmm.posteriors(m, rng.normal(size=12), include_xi=True)
    assert fb.xi.shape == (11, 3, 3)
    for t in range(11):
        assert fb.xi[t].sum() == pytest.approx(1.0, abs=1e-9)
        assert np.allclose(fb.xi[t].sum(axis=1), fb.gamma[t], atol=1e-9)
    m_u = loghmm.HmmModel([1.0], [[1.0]], (loghmm.Uniform(0.0, 1.0),))
    with pytest.raises(loghmm.InfeasibleSequenceError, match="impossible"):
        loghmm.posteriors(m_u, [0.5, 3.0])
    with pytest.raises(loghmm.InfeasibleSequenceError, match="feasible"):
        loghmm.viterbi(m_u, [5.0])
    rng = np.random.default_rng(9)
    for _ in range(100):
        k = int(rng.integers(1, 4))
        m = rand_gauss(loghmm, rng, k)
        seq = rng.normal(size=int(rng.integers(1, 15)))
        res = loghmm.viterbi(m, seq)
        _, ll = loghmm.forward_log(m, seq)
        assert res.log_joint <= ll + 1e-12
        ref = orig["viterbi"](m, seq)
        assert np.array_equal(res.path, ref.path) and res.log_joint == ref.log_joint
    sym = loghmm.HmmModel([0.5, 0.5], [[0.7, 0.3], [0.3, 0.7]],
                          (loghmm.Gaussian(-1.0, 0.8), loghmm.Gaussian(1.0, 1.3)))
    seq = np.random.default_rng(12).normal(size=25)
    assert loghmm.forward_log(sym, seq)[1] == pytest.approx(loghmm.forward_log(sym, seq[::-1])[1], abs=1e-9)
    with pytest.raises(ValueError, match="NaN"):
        loghmm.posteriors(sym, [0.1, float("nan")])


def test_training_through_the_reference_api(L):
    """test_training.py TestCollapseGuard / TestMultiSequence through the shim:
    reference objects in, reference objects out, reference errors."""
    loghmm, orig = L
    frozen = loghmm.Gaussian(42.0, 7.0)
    model = loghmm.HmmModel([1.0, 0.0], [[1.0, 0.0], [0.0, 1.0]], (loghmm.Gaussian(0.0, 1.0), frozen))
    seq = np.random.default_rng(5).normal(size=60)
    cfg = loghmm.TrainingConfig(max_iterations=10)
    fitted, report = loghmm.baum_welch(model, [seq], cfg)
    ref_fit, ref_rep = orig["baum_welch"](model, [seq], cfg)
    assert type(fitted) is loghmm.HmmModel and type(report) is loghmm.training.TrainingReport
    assert fitted.emissions[1] is frozen
    assert report.collapsed_states == ref_rep.collapsed_states
    np.testing.assert_allclose(report.log_likelihood_trace, ref_rep.log_likelihood_trace, rtol=1e-12)
    assert fitted.emissions[0].mu == pytest.approx(ref_fit.emissions[0].mu, rel=1e-12)
    rng = np.random.default_rng(8)
    s1, s2 = rng.normal(0, 1, 30), rng.normal(2, 1, 45)
    init = loghmm.training.default_initial_model(2, "gaussian", [s1, s2])
    fitted, rep = loghmm.baum_welch(init, [s1, s2], loghmm.TrainingConfig(max_iterations=20))
    _, l1 = loghmm.forward_log(fitted, s1)
    _, l2 = loghmm.forward_log(fitted, s2)
    assert rep.log_likelihood_trace[-1] == pytest.approx(l1 + l2, abs=1e-9)
    with pytest.raises(loghmm.TrainingError):
        loghmm.baum_welch(loghmm.HmmModel([1.0], [[1.0]], (loghmm.Gaussian(0, 1),)), [])
    m_u = loghmm.HmmModel([0.5, 0.5], [[0.5, 0.5], [0.5, 0.5]],
                          (loghmm.Uniform(0.0, 1.0), loghmm.Uniform(0.5, 2.0)))
    with pytest.raises(loghmm.TrainingError, match=r"sequence 1, index 2"):
        loghmm.baum_welch(m_u, [np.array([0.5, 0.7]), np.array([0.5, 0.7, 9.0])])
    sc, sr = loghmm.score_model(fitted, [s1, s2]), orig["score_model"](fitted, [s1, s2])
    assert type(sc) is loghmm.training.ModelScore
    assert sc.log_likelihood == pytest.approx(sr.log_likelihood, rel=1e-12) and sc.num_params == sr.num_params
