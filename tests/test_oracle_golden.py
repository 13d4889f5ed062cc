"""Pin the CPU oracle (oracle/loghmm_oracle.py) against the reference's own
golden vectors (tests/golden/, produced by tests/golden/make_golden.py from
the unmodified reference) -- CPU only."""

import math

import numpy as np
import pytest

import loghmm_oracle as O


def tables(case):
    lp, la = O.model_tables(case["pi"], case["A"])
    return lp, la


def fams(case):
    return [tuple(e) for e in case["emissions"]]


def test_emission_matrix(golden):
    for c in golden["cases"]:
        y = golden["vec"][c["name"] + "_y"]
        lb = O.emission_matrix(fams(c), y)
        ref = golden["vec"][c["name"] + "_logb"]
        if c["family"] in ("gaussian", "poisson"):
            # IEEE-basic-op families: bit-exact
            assert np.array_equal(lb, ref), c["name"]
        else:
            np.testing.assert_allclose(lb, ref, rtol=1e-13, atol=1e-13, err_msg=c["name"])


def test_forward_backward(golden):
    for c in golden["cases"]:
        v = golden["vec"]
        y = v[c["name"] + "_y"]
        lp, la = tables(c)
        r = O.posteriors(lp, la, O.emission_matrix(fams(c), y), include_xi=True)
        assert r["ll"] == pytest.approx(c["ll"], rel=1e-13, abs=1e-12)
        np.testing.assert_allclose(r["log_alpha"], v[c["name"] + "_log_alpha"], rtol=1e-13, atol=1e-11)
        np.testing.assert_allclose(r["log_beta"], v[c["name"] + "_log_beta"], rtol=1e-13, atol=1e-11)
        np.testing.assert_allclose(r["gamma"], v[c["name"] + "_gamma"], atol=1e-12)
        np.testing.assert_allclose(r["xi"], v[c["name"] + "_xi"], atol=1e-12)


def test_viterbi_exact(golden):
    for c in golden["cases"]:
        v = golden["vec"]
        y = v[c["name"] + "_y"]
        lp, la = tables(c)
        path, lj, back = O.viterbi(lp, la, O.emission_matrix(fams(c), y))
        assert np.array_equal(path, v[c["name"] + "_path"]), c["name"]
        if c["family"] in ("gaussian", "poisson"):
            assert lj == c["log_joint"]
        else:
            assert lj == pytest.approx(c["log_joint"], rel=1e-13)
        assert (back[0] == 0).all()


def test_baum_welch_short(golden):
    v = golden["vec"]
    for c in golden["cases"]:
        y = v[c["name"] + "_y"]
        pi, A, em, trace, conv, coll = O.baum_welch(c["pi"], c["A"], fams(c), [y, y[::-1].copy()],
                                                    c["bw"]["max_iterations"])
        np.testing.assert_allclose(trace, c["bw"]["trace"], rtol=1e-12)
        np.testing.assert_allclose(pi, v[c["name"] + "_bw_pi"], atol=1e-12)
        np.testing.assert_allclose(A, v[c["name"] + "_bw_A"], atol=1e-12)
        for a, b in zip(em, c["bw"]["emissions"]):
            assert a[0] == b[0]
            np.testing.assert_allclose(a[1:], b[1:], rtol=1e-10)


def test_config1(golden):
    v, c1 = golden["vec"], golden["c1"]
    y = v["c1_y"]
    em = [("gaussian", -0.5, 1.0), ("gaussian", 1.5, 1.0)]
    lp, la = O.model_tables([0.5, 0.5], [[0.9, 0.1], [0.1, 0.9]])
    lb = O.emission_matrix(em, y)
    r = O.posteriors(lp, la, lb)
    assert r["ll"] == pytest.approx(c1["ll"], rel=1e-14)
    np.testing.assert_allclose(r["gamma"], v["c1_gamma"], atol=1e-13)
    path, lj, _ = O.viterbi(lp, la, lb)
    assert np.array_equal(path, v["c1_path"]) and lj == c1["log_joint"]
    pi, A, emf, trace, _, _ = O.baum_welch([0.5, 0.5], [[0.9, 0.1], [0.1, 0.9]], em, [y], 2)
    np.testing.assert_allclose(trace, c1["bw_trace"], rtol=1e-13)
    np.testing.assert_allclose(A, c1["bw_A"], atol=1e-13)


def test_frontend_earthquake(golden):
    eq = golden["front"]["earthquake"]
    y = np.array(eq["observations"], dtype=float)
    exp = eq["expected"]
    # default_initial_model(2, "poisson", ...) (training.py:239-282): sorted quantile bins
    pooled = np.sort(y)
    bins = np.array_split(pooled, 2)
    em = [("poisson", max(float(b.mean()), 1e-9)) for b in bins]
    pi, A, emf, trace, conv, _ = O.baum_welch([0.5, 0.5], [[0.9, 0.1], [0.1, 0.9]], em, [y], 500,
                                              rel_tol=1e-8)
    assert conv and len(trace) == exp["iterations"]
    assert trace[-1] == pytest.approx(exp["log_likelihood"], abs=1e-10)
    assert sorted(e[1] for e in emf) == pytest.approx(exp["rates_sorted"], rel=1e-12)
    lp, la = O.model_tables(pi, A)
    lb = O.emission_matrix(emf, y)
    path, _, _ = O.viterbi(lp, la, lb)
    assert path.tolist() == exp["viterbi_path"]
    r = O.posteriors(lp, la, lb)
    assert np.argmax(r["gamma"], axis=1).tolist() == exp["posterior_path"]


def test_frontend_small(golden):
    for case in golden["front"]["small_models"]:
        doc = case["model_document"]
        em = [("gaussian", e["params"]["mu"], e["params"]["sigma"]) for e in doc["emissions"]]
        y = np.array(case["observations"], dtype=float)
        lp, la = O.model_tables(doc["initial"], doc["transitions"])
        lb = O.emission_matrix(em, y)
        r = O.posteriors(lp, la, lb)
        assert r["ll"] == pytest.approx(case["expected"]["log_likelihood"], abs=1e-12)
        assert O.viterbi(lp, la, lb)[0].tolist() == case["expected"]["viterbi_path"]
        assert np.argmax(r["gamma"], axis=1).tolist() == case["expected"]["posterior_path"]


def test_fp32_viterbi_restatement_consistency():
    """The fp32 restatement follows the fp64 path ordering: on a well
    separated model the decoded paths agree."""
    rng = np.random.default_rng(3)
    y = np.concatenate([rng.normal(-3, 0.5, 50), rng.normal(3, 0.5, 50)])
    em = [("gaussian", -3.0, 0.5), ("gaussian", 3.0, 0.5)]
    lp, la = O.model_tables([0.5, 0.5], [[0.9, 0.1], [0.1, 0.9]])
    p64 = O.viterbi(lp, la, O.emission_matrix(em, y))[0]
    p32 = O.viterbi(lp, la, O.emission_matrix(em, y.astype(np.float32), np.float32), np.float32)[0]
    assert np.array_equal(p64, p32)


def test_special_functions_against_mpmath():
    mpmath = pytest.importorskip("mpmath")
    for x in (0.3, 1.0, 2.5, 7.0, 15.0, 120.0):
        assert O.digamma(x) == pytest.approx(float(mpmath.digamma(x)), rel=1e-12)
        assert O.trigamma(x) == pytest.approx(float(mpmath.polygamma(1, x)), rel=1e-11)
    for k in (0.1, 1.0, 3.7, 3.8, 20.0):
        assert O.i1_i0_ratio(k) == pytest.approx(float(mpmath.besseli(1, k) / mpmath.besseli(0, k)), abs=2e-7)
        assert O.log_bessel_i0(k) == pytest.approx(float(mpmath.log(mpmath.besseli(0, k))), abs=2e-7)
