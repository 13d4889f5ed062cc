"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle and
the reference's golden vectors.

Tolerances (BASELINE.json north_star):
  fp64: LL / params <= 1e-9 relative, posteriors <= 1e-9 absolute
  fp32: LL <= 1e-4 relative, posteriors <= 1e-5 absolute
  Viterbi paths / backpointers: bit-exact (fp64 vs the reference for the
  IEEE-basic-op families Gaussian and Poisson; fp32 vs the fp32 restatement);
  for Student-t / Gamma / von Mises the emission calls log1p/log/cos whose
  last ulp differs between CUDA and numpy, so a differing backpointer is only
  accepted at a near-tie (candidate gap within 64 ulps of the score).
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import loghmm_oracle as O  # noqa: E402

import paper_2605_29208_b200 as H  # noqa: E402
from paper_2605_29208_b200 import engine  # noqa: E402
from paper_2605_29208_b200.configs import make_config  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def to_model(pi, A, ems):
    d = []
    for e in ems:
        k = e[0]
        if k == "gaussian":
            d.append(H.Gaussian(e[1], e[2]))
        elif k == "student_t":
            d.append(H.StudentT(e[1], e[2], e[3]))
        elif k == "gamma":
            d.append(H.Gamma(e[1], e[2]))
        elif k == "von_mises":
            d.append(H.VonMises(e[1], e[2]))
        elif k == "poisson":
            d.append(H.Poisson(e[1]))
        elif k == "joint":
            d.append(H.Joint(to_model([1.0], [[1.0]], [e[1]]).emissions[0],
                             to_model([1.0], [[1.0]], [e[2]]).emissions[0]))
    return H.HmmModel(pi, A, tuple(d))


def to_tuples(model):
    out = []
    for d in model.emissions:
        if isinstance(d, H.Joint):
            out.append(("joint", to_tuples(H.HmmModel([1.0], [[1.0]], (d.first,)))[0],
                        to_tuples(H.HmmModel([1.0], [[1.0]], (d.second,)))[0]))
        else:
            out.append((d.family,) + tuple(d.params().values()))
    return out


EXACT_FAMS = ("gaussian", "poisson")


def test_emission_matches_reference(golden):
    for c in golden["cases"]:
        m = to_model(c["pi"], c["A"], c["emissions"])
        y = golden["vec"][c["name"] + "_y"]
        lb = H.emission_log_matrix(m, y)
        ref = golden["vec"][c["name"] + "_logb"]
        if c["family"] in EXACT_FAMS:
            assert np.array_equal(lb, ref), c["name"]
        else:
            np.testing.assert_allclose(lb, ref, rtol=1e-13, atol=1e-13, err_msg=c["name"])


def test_posteriors_match_reference(golden):
    v = golden["vec"]
    for c in golden["cases"]:
        m = to_model(c["pi"], c["A"], c["emissions"])
        y = v[c["name"] + "_y"]
        fb = H.posteriors(m, y, include_xi=True)
        assert fb.log_likelihood == pytest.approx(c["ll"], rel=1e-9), c["name"]
        np.testing.assert_allclose(fb.gamma, v[c["name"] + "_gamma"], atol=1e-9, err_msg=c["name"])
        np.testing.assert_allclose(fb.log_alpha, v[c["name"] + "_log_alpha"], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(fb.log_beta, v[c["name"] + "_log_beta"], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(fb.xi, v[c["name"] + "_xi"], atol=1e-9, err_msg=c["name"])
        np.testing.assert_allclose(fb.gamma.sum(axis=1), 1.0, atol=1e-12)


def _near_tie_ok(lp, la, lb, t, j, ours, theirs, dtype=np.float64):
    """Backpointer disagreement is allowed only at a near-tie of the two
    candidates (|gap| within 64 ulps of the score magnitude)."""
    # recompute the oracle's score at t-1 in the same precision
    R = dtype
    score = np.asarray(lp, R) + np.asarray(lb[0], R)
    for s in range(1, t):
        cand = score[:, None] + np.asarray(la, R)
        score = cand[np.argmax(cand, axis=0), np.arange(len(score))] + np.asarray(lb[s], R)
    cand = score[:, None] + np.asarray(la, R)
    gap = abs(float(cand[ours, j]) - float(cand[theirs, j]))
    return gap <= 64 * np.finfo(R).eps * max(1.0, abs(float(cand[theirs, j])))


def test_viterbi_matches_reference(golden, vit_algo):
    v = golden["vec"]
    for c in golden["cases"]:
        m = to_model(c["pi"], c["A"], c["emissions"])
        y = v[c["name"] + "_y"]
        res = H.viterbi(m, y)
        bv = H.viterbi_batch(m, y, back=True)
        back = bv.back.cpu().numpy().astype(np.int64)
        lp, la = O.model_tables(c["pi"], c["A"])
        lbm = v[c["name"] + "_logb"]
        opath, olj, oback = O.viterbi(lp, la, lbm)
        if c["family"] in EXACT_FAMS:
            assert np.array_equal(res.path, v[c["name"] + "_path"]), c["name"]
            assert res.log_joint == c["log_joint"], c["name"]
            assert np.array_equal(back, oback), c["name"]
        else:
            diff = np.argwhere(back != oback)
            for t, j in diff:
                assert _near_tie_ok(lp, la, lbm, t, j, back[t, j], oback[t, j]), (c["name"], t, j)
            if diff.size == 0:
                assert np.array_equal(res.path, v[c["name"] + "_path"])
            assert res.log_joint == pytest.approx(c["log_joint"], rel=1e-12)


def _random_gauss_model(rng, K):
    pi = rng.dirichlet(np.ones(K))
    A = rng.dirichlet(np.ones(K), size=K) * 0.4 + 0.6 * np.eye(K)
    A /= A.sum(1, keepdims=True)
    return H.HmmModel(pi, A, tuple(H.Gaussian(float(rng.normal(0, 2)), float(rng.uniform(0.4, 1.5)))
                                   for _ in range(K)))


@pytest.fixture(params=["auto", "chain", "lanes"])
def vit_algo(request, monkeypatch):
    """Run a test under every Viterbi layout: the automatic choice (K lanes per
    sequence for Gaussian / Poisson, the chain-warp kernel for the families
    with transcendental densities at K <= 4) and each layout forced."""
    if request.param != "auto":
        monkeypatch.setenv("LOGHMM_VIT_ALGO", request.param)
    else:
        monkeypatch.delenv("LOGHMM_VIT_ALGO", raising=False)
    return request.param


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("T", [4, 8, 36, 1000, 1024])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_viterbi_equal_length_bitexact(K, T, dtype, vit_algo):
    """Equal-length batches: path, backpointers and log joint bit-identical
    to the reference restatement, including exact ties (a model with a
    duplicated state, so candidates tie every step and the first index must
    win)."""
    rng = np.random.default_rng(1000 * K + T)
    m = _random_gauss_model(rng, K)
    if K >= 3:  # duplicate state 0 into state 2: candidate ties every step
        mus = [d.mu for d in m.emissions]
        sds = [d.sigma for d in m.emissions]
        mus[2], sds[2] = mus[0], sds[0]
        A = np.array(m.transitions)
        A[2, :] = A[0, :]
        A[:, 2] = A[:, 0]
        A /= A.sum(1, keepdims=True)
        pi = np.array(m.initial)
        pi[2] = pi[0]
        pi /= pi.sum()
        m = H.HmmModel(pi, A, tuple(H.Gaussian(a, b) for a, b in zip(mus, sds)))
    seqs = [rng.normal(0, 3, T) for _ in range(37)]
    out = H.viterbi_batch(m, seqs, dtype=dtype, back=True)
    path = out.path.cpu().numpy()
    back = out.back.cpu().numpy()
    lj = out.log_joint.cpu().numpy()
    lp, la = O.model_tables(m.initial, m.transitions)
    R = np.float32 if dtype == "float32" else np.float64
    for b, y in enumerate(seqs):
        yy = y.astype(R)
        lb = O.emission_matrix(to_tuples(m), yy, R)
        p, j, bk = O.viterbi(lp.astype(R), la.astype(R), lb, R)
        s = slice(b * T, (b + 1) * T)
        assert np.array_equal(path[s], p), (K, T, b)
        assert np.array_equal(back[s].astype(np.int64), bk), (K, T, b)
        assert lj[b] == j


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5, 8])
def test_fp32_viterbi_bitexact_ragged(K, vit_algo):
    rng = np.random.default_rng(100 + K)
    m = _random_gauss_model(rng, K)
    lens = [1, 2, 31, 32, 33, 64, 100, 257, 1024, 700]
    seqs = [rng.normal(0, 3, n) for n in lens]
    out = H.viterbi_batch(m, seqs, dtype="float32", back=True)
    path = out.path.cpu().numpy()
    back = out.back.cpu().numpy()
    lj = out.log_joint.cpu().numpy()
    lp, la = O.model_tables(m.initial, m.transitions)
    off = out.offsets
    for b, y in enumerate(seqs):
        lb32 = O.emission_matrix(to_tuples(m), y.astype(np.float32), np.float32)
        p, j, bk = O.viterbi(lp.astype(np.float32), la.astype(np.float32), lb32, np.float32)
        assert np.array_equal(path[off[b]:off[b + 1]], p), (K, b)
        assert np.array_equal(back[off[b]:off[b + 1]], bk), (K, b)
        assert lj[b] == j


@pytest.mark.parametrize("K", [2, 3, 4, 7])
def test_fp64_viterbi_poisson_bitexact(K, vit_algo):
    rng = np.random.default_rng(7 + K)
    pi = rng.dirichlet(np.ones(K))
    A = rng.dirichlet(np.ones(K), size=K)
    m = H.HmmModel(pi, A, tuple(H.Poisson(float(r)) for r in rng.uniform(0.5, 20, K)))
    seqs = [rng.poisson(8.0, n).astype(float) for n in (5, 77, 300, 1500)]
    out = H.viterbi_batch(m, seqs, back=True)
    lp, la = O.model_tables(pi, A)
    for b, y in enumerate(seqs):
        p, j, bk = O.viterbi(lp, la, O.emission_matrix(to_tuples(m), y))
        s = slice(out.offsets[b], out.offsets[b + 1])
        assert np.array_equal(out.path.cpu().numpy()[s], p)
        assert np.array_equal(out.back.cpu().numpy()[s].astype(np.int64), bk)
        assert out.log_joint.cpu().numpy()[b] == j


@pytest.fixture(params=["chunked", "auto"])
def fb_algo(request, monkeypatch):
    """Run a test under both forward-backward decompositions: the chunked scan
    (forced) and the automatic choice, which takes the chunk-operator +
    meet-in-the-middle kernel for equal-length batches."""
    if request.param == "chunked":
        monkeypatch.setenv("LOGHMM_FB_ALGO", "chunked")
    else:
        monkeypatch.delenv("LOGHMM_FB_ALGO", raising=False)
    return request.param


@pytest.mark.parametrize("K", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("T", [8, 64, 1000, 1024])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_posteriors_equal_length(K, T, dtype, fb_algo):
    """Equal-length batches (the [B, T] layout of the BASELINE configs) under
    both decompositions against the oracle: LL, gamma, log alpha, log beta."""
    rng = np.random.default_rng(100 * K + T)
    m = _random_gauss_model(rng, K)
    seqs = [rng.normal(0, 3, T) for _ in range(5)]
    r = H.posteriors_batch(m, seqs, dtype=dtype)
    lp, la = O.model_tables(m.initial, m.transitions)
    g = r.gamma.cpu().numpy().astype(np.float64)
    A_ = r.log_alpha.cpu().numpy().astype(np.float64)
    B_ = r.log_beta.cpu().numpy().astype(np.float64)
    ll = r.log_likelihood.cpu().numpy()
    for b, y in enumerate(seqs):
        yy = y.astype(np.float32).astype(np.float64) if dtype == "float32" else y
        o = O.posteriors(lp, la, O.emission_matrix(to_tuples(m), yy))
        s = slice(b * T, (b + 1) * T)
        if dtype == "float64":
            assert ll[b] == pytest.approx(o["ll"], rel=1e-9)
            np.testing.assert_allclose(g[s], o["gamma"], atol=1e-9)
            np.testing.assert_allclose(A_[s], o["log_alpha"], rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(B_[s], o["log_beta"], rtol=1e-9, atol=1e-9)
        else:
            assert ll[b] == pytest.approx(o["ll"], rel=1e-4)
            np.testing.assert_allclose(g[s], o["gamma"], atol=1e-5)
            np.testing.assert_allclose(A_[s], o["log_alpha"], rtol=1e-5, atol=1e-3)
            np.testing.assert_allclose(B_[s], o["log_beta"], rtol=1e-5, atol=1e-3)


def _estep_partials(model, data, dtype, algo, monkeypatch):
    if algo == "chunked":
        monkeypatch.setenv("LOGHMM_FB_ALGO", "chunked")
    else:
        monkeypatch.delenv("LOGHMM_FB_ALGO", raising=False)
    dm = engine.DeviceModel.from_model(model)
    batch = engine.make_batch(data, model.n_streams, dtype)
    o = engine.forward_backward(batch, dm, stats=True)
    return o.partials.cpu().numpy(), o.ll.cpu().numpy(), o.flags.cpu().numpy()


@pytest.mark.parametrize("name,B,T", [("c2", 6, 1024), ("c3", 4, 2048), ("c4", 4, 2000),
                                      ("pois4", 4, 512)])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_estep_statistics_both_decompositions(name, B, T, dtype, monkeypatch):
    """Per-sequence E-step statistics (xi totals, gamma totals, gamma_0, family
    sums) of the meet-in-the-middle kernel equal the chunked scan's, for every
    family configuration it serves (Gaussian, Student-t, Gamma+von Mises,
    Poisson)."""
    if name == "pois4":
        rng = np.random.default_rng(3)
        K = 4
        A = rng.dirichlet(np.ones(K), size=K) * 0.3 + 0.7 * np.eye(K)
        A /= A.sum(1, keepdims=True)
        model = H.HmmModel(np.full(K, 1 / K), A, tuple(H.Poisson(0.5 * (k + 1)) for k in range(K)))
        data = [rng.poisson(2.0, T).astype(np.float64) for _ in range(B)]
    else:
        cfg = make_config(name, B=B, T=T)
        model = cfg.init
        data = [cfg.data[b] for b in range(B)]
    pa, la, fa = _estep_partials(model, data, dtype, "auto", monkeypatch)
    pc, lc, fc = _estep_partials(model, data, dtype, "chunked", monkeypatch)
    rt = 1e-9 if dtype == "float64" else 2e-4
    np.testing.assert_allclose(la, lc, rtol=rt)
    np.testing.assert_array_equal(fa, fc)
    scale = np.abs(pc).max(axis=1, keepdims=True) + 1e-300
    np.testing.assert_allclose(pa / scale, pc / scale, atol=rt * 10)


@pytest.mark.parametrize("K", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_posteriors_batch_ragged(K, dtype, fb_algo):
    rng = np.random.default_rng(11 * K)
    m = _random_gauss_model(rng, K)
    lens = [1, 2, 5, 31, 32, 33, 100, 1000, 1025]
    seqs = [rng.normal(0, 3, n) for n in lens]
    r = H.posteriors_batch(m, seqs, dtype=dtype, include_xi=True)
    lp, la = O.model_tables(m.initial, m.transitions)
    g = r.gamma.cpu().numpy().astype(np.float64)
    A_ = r.log_alpha.cpu().numpy().astype(np.float64)
    B_ = r.log_beta.cpu().numpy().astype(np.float64)
    X_ = r.xi.cpu().numpy().astype(np.float64)
    ll = r.log_likelihood.cpu().numpy()
    for b, y in enumerate(seqs):
        yy = y.astype(np.float32).astype(np.float64) if dtype == "float32" else y
        o = O.posteriors(lp, la, O.emission_matrix(to_tuples(m), yy), include_xi=True)
        s = slice(r.offsets[b], r.offsets[b + 1])
        xs = slice(r.offsets[b] - b, r.offsets[b + 1] - b - 1)
        if dtype == "float64":
            assert ll[b] == pytest.approx(o["ll"], rel=1e-9)
            np.testing.assert_allclose(g[s], o["gamma"], atol=1e-9)
            np.testing.assert_allclose(A_[s], o["log_alpha"], rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(B_[s], o["log_beta"], rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(X_[xs], o["xi"], atol=1e-9)
        else:
            assert ll[b] == pytest.approx(o["ll"], rel=1e-4)
            np.testing.assert_allclose(g[s], o["gamma"], atol=1e-5)
            np.testing.assert_allclose(A_[s], o["log_alpha"], rtol=1e-5, atol=1e-3)
            np.testing.assert_allclose(B_[s], o["log_beta"], rtol=1e-5, atol=1e-3)
            np.testing.assert_allclose(X_[xs], o["xi"], atol=1e-5)


def test_baum_welch_matches_reference(golden, fb_algo):
    v = golden["vec"]
    for c in golden["cases"]:
        m = to_model(c["pi"], c["A"], c["emissions"])
        y = v[c["name"] + "_y"]
        cfg = H.TrainingConfig(max_iterations=c["bw"]["max_iterations"], rel_tol=1e-300)
        fitted, rep = H.baum_welch(m, [y, y[::-1].copy()], cfg)
        np.testing.assert_allclose(rep.log_likelihood_trace, c["bw"]["trace"], rtol=1e-9, err_msg=c["name"])
        np.testing.assert_allclose(fitted.initial, v[c["name"] + "_bw_pi"], atol=1e-9)
        np.testing.assert_allclose(fitted.transitions, v[c["name"] + "_bw_A"], atol=1e-9)
        for a, b in zip(to_tuples(fitted), c["bw"]["emissions"]):
            assert a[0] == b[0]
            np.testing.assert_allclose(a[1:], b[1:], rtol=1e-8, err_msg=c["name"])
        assert [list(x) for x in rep.collapsed_states] == c["bw"]["collapsed"]


def test_config1(golden):
    v, c1 = golden["vec"], golden["c1"]
    cfg = make_config("c1")
    y = cfg.data[0]
    assert np.array_equal(y, v["c1_y"])
    fb = H.posteriors(cfg.init, y)
    assert fb.log_likelihood == pytest.approx(c1["ll"], rel=1e-12)
    np.testing.assert_allclose(fb.gamma, v["c1_gamma"], atol=1e-10)
    vit = H.viterbi(cfg.init, y)
    assert np.array_equal(vit.path, v["c1_path"]) and vit.log_joint == c1["log_joint"]
    fitted, rep = H.baum_welch(cfg.init, [y], H.TrainingConfig(max_iterations=2, rel_tol=1e-300))
    np.testing.assert_allclose(rep.log_likelihood_trace, c1["bw_trace"], rtol=1e-12)
    np.testing.assert_allclose(fitted.transitions, c1["bw_A"], atol=1e-10)
    for a, b in zip(to_tuples(fitted), c1["bw_emissions"]):
        np.testing.assert_allclose(a[1:], b[1:], rtol=1e-9)


def test_earthquake_fixture(golden):
    eq = golden["front"]["earthquake"]
    y = np.array(eq["observations"], dtype=float)
    exp = eq["expected"]
    start = H.default_initial_model(2, "poisson", [y])
    fitted, rep = H.baum_welch(start, [y])
    assert rep.converged and rep.iterations == exp["iterations"]
    assert rep.log_likelihood_trace[-1] == pytest.approx(exp["log_likelihood"], abs=1e-9)
    assert sorted(d.rate for d in fitted.emissions) == pytest.approx(exp["rates_sorted"], rel=1e-9)
    assert H.viterbi(fitted, y).path.tolist() == exp["viterbi_path"]
    assert H.posterior_decode(H.posteriors(fitted, y)).tolist() == exp["posterior_path"]
    sc = H.score_model(fitted, [y])
    assert sc.log_likelihood == pytest.approx(exp["score"]["log_likelihood"], abs=1e-9)
    assert sc.num_params == exp["score"]["num_params"]


def test_small_model_fixtures(golden):
    for case in golden["front"]["small_models"]:
        doc = case["model_document"]
        m = to_model(doc["initial"], doc["transitions"],
                     [("gaussian", e["params"]["mu"], e["params"]["sigma"]) for e in doc["emissions"]])
        y = np.array(case["observations"], dtype=float)
        fb = H.posteriors(m, y)
        assert fb.log_likelihood == pytest.approx(case["expected"]["log_likelihood"], abs=1e-12)
        assert H.viterbi(m, y).path.tolist() == case["expected"]["viterbi_path"]
        assert H.posterior_decode(fb).tolist() == case["expected"]["posterior_path"]


def test_underflow_100k(golden):
    u = golden["underflow"]
    rng = np.random.default_rng(7)
    m = H.HmmModel([0.5, 0.5], [[0.97, 0.03], [0.05, 0.95]], (H.Gaussian(0.0, 1.0), H.Gaussian(2.5, 1.8)))
    seq = rng.normal(size=100_000) * 2.0 + 1.0
    fb = H.posteriors(m, seq)
    assert fb.log_likelihood == pytest.approx(u["ll"], rel=1e-9)
    np.testing.assert_allclose(fb.gamma[0], u["gamma_row0"], atol=1e-9)
    np.testing.assert_allclose(fb.gamma[-1], u["gamma_last"], atol=1e-9)
    assert np.abs(fb.gamma.sum(axis=1) - 1.0).max() < 1e-6
    assert H.viterbi(m, seq).log_joint == u["viterbi_log_joint"]
    fb32 = H.posteriors(m, seq, dtype="float32")
    assert fb32.log_likelihood == pytest.approx(u["ll"], rel=1e-4)


def test_error_semantics():
    m = H.HmmModel([0.5, 0.5], [[0.5, 0.5], [0.5, 0.5]], (H.Poisson(2.0), H.Poisson(5.0)))
    with pytest.raises(H.InfeasibleSequenceError, match="sequence impossible under model"):
        H.posteriors(m, np.array([1.0, 2.5, 3.0]))
    with pytest.raises(H.InfeasibleSequenceError, match="no feasible path"):
        H.viterbi(m, np.array([1.0, 2.5, 3.0]))
    with pytest.raises(H.TrainingError, match="sequence 1, index 2"):
        H.baum_welch(m, [np.array([1.0, 2.0]), np.array([1.0, 2.0, 0.5])],
                     H.TrainingConfig(max_iterations=2))
    with pytest.raises(ValueError, match="NaN"):
        H.posteriors(m, np.array([1.0, np.nan]))
    with pytest.raises(ValueError, match="non-empty"):
        H.posteriors(m, np.array([]))


def test_single_state_and_single_step():
    m = H.HmmModel([1.0], [[1.0]], (H.Gaussian(0.3, 1.7),))
    y = np.array([0.1, -2.0, 3.3])
    fb = H.posteriors(m, y)
    assert fb.log_likelihood == pytest.approx(float(O.emission_matrix([("gaussian", 0.3, 1.7)], y).sum()), rel=1e-12)
    m2 = _random_gauss_model(np.random.default_rng(1), 3)
    fb1 = H.posteriors(m2, np.array([0.4]))
    lp, la = O.model_tables(m2.initial, m2.transitions)
    o = O.posteriors(lp, la, O.emission_matrix(to_tuples(m2), np.array([0.4])))
    assert fb1.log_likelihood == pytest.approx(o["ll"], rel=1e-12)
    assert np.array_equal(fb1.log_beta, np.zeros((1, 3)))


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_config2_full_size(dtype):
    """BASELINE config 2 at full size (B=4096, T=1024): size-independent
    properties on all sequences, oracle parity on a seeded subset."""
    cfg = make_config("c2")
    model = cfg.init
    r = H.posteriors_batch(model, cfg.data, dtype=dtype)
    vit = H.viterbi_batch(model, cfg.data, dtype=dtype)
    g = r.gamma.double()
    assert torch.isfinite(r.log_likelihood).all()
    assert (g.sum(dim=1) - 1).abs().max().item() < (1e-12 if dtype == "float64" else 1e-5)
    assert (vit.log_joint <= r.log_likelihood + 1e-6 * r.log_likelihood.abs()).all()
    rng = np.random.default_rng(5)
    lp, la = O.model_tables(model.initial, model.transitions)
    T = cfg.T
    for b in rng.choice(cfg.B, 6, replace=False):
        y = cfg.data[b]
        yy = y.astype(np.float32).astype(np.float64) if dtype == "float32" else y
        o = O.posteriors(lp, la, O.emission_matrix(to_tuples(model), yy))
        s = slice(b * T, (b + 1) * T)
        tol_ll, tol_g = (1e-9, 1e-9) if dtype == "float64" else (1e-4, 1e-5)
        assert r.log_likelihood[b].item() == pytest.approx(o["ll"], rel=tol_ll)
        np.testing.assert_allclose(r.gamma[s].double().cpu().numpy(), o["gamma"], atol=tol_g)
        if dtype == "float64":
            p, j, _ = O.viterbi(lp, la, O.emission_matrix(to_tuples(model), y))
        else:
            p, j, _ = O.viterbi(lp.astype(np.float32), la.astype(np.float32),
                                O.emission_matrix(to_tuples(model), y.astype(np.float32), np.float32),
                                np.float32)
        assert np.array_equal(vit.path[s].cpu().numpy(), p)
        assert vit.log_joint[b].item() == j


@pytest.mark.parametrize("name,B,T,iters", [("c2", 48, 1024, 3), ("c3", 16, 2048, 3),
                                            ("c4", 12, 2000, 3), ("c5", 2, 4096, 2)])
def test_config_baum_welch_subset(name, B, T, iters, fb_algo):
    """Baum-Welch parity on a seeded subset of each BASELINE config."""
    cfg = make_config(name, B=B, T=T)
    data = [cfg.data[b] for b in range(B)]
    fitted, rep = H.baum_welch(cfg.init, data, H.TrainingConfig(max_iterations=iters, rel_tol=1e-300))
    pi, A, em, trace, _, _ = O.baum_welch(cfg.init.initial, cfg.init.transitions, to_tuples(cfg.init),
                                          data, iters)
    np.testing.assert_allclose(rep.log_likelihood_trace, trace, rtol=1e-9)
    np.testing.assert_allclose(fitted.transitions, A, atol=1e-9)
    np.testing.assert_allclose(fitted.initial, pi, atol=1e-9)
    for a, b in zip(to_tuples(fitted), em):
        if a[0] == "joint":
            np.testing.assert_allclose(a[1][1:], b[1][1:], rtol=1e-8)
            np.testing.assert_allclose(a[2][1:], b[2][1:], rtol=1e-8)
        else:
            np.testing.assert_allclose(a[1:], b[1:], rtol=1e-8)


def test_config5_viterbi_and_posteriors_subset():
    cfg = make_config("c5", B=2, T=3000)
    model = cfg.truth
    lp, la = O.model_tables(model.initial, model.transitions)
    r = H.posteriors_batch(model, cfg.data)
    vit = H.viterbi_batch(model, cfg.data, back=True)
    for b in range(2):
        lb = O.emission_matrix(to_tuples(model), cfg.data[b])
        o = O.posteriors(lp, la, lb)
        s = slice(b * cfg.T, (b + 1) * cfg.T)
        assert r.log_likelihood[b].item() == pytest.approx(o["ll"], rel=1e-9)
        np.testing.assert_allclose(r.gamma[s].cpu().numpy(), o["gamma"], atol=1e-9)
        p, j, bk = O.viterbi(lp, la, lb)
        assert np.array_equal(vit.path[s].cpu().numpy(), p)
        assert np.array_equal(vit.back[s].cpu().numpy().astype(np.int64), bk)
        assert vit.log_joint[b].item() == j


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_exact_gaussian_emission_wide_range(dtype):
    """The hoisted-reciprocal division in the exact emission reproduces the
    reference's IEEE quotient (hence log b) bit for bit over a wide range of
    magnitudes, including values that underflow or overflow the square."""
    rng = np.random.default_rng(17)
    R = np.float64 if dtype == "float64" else np.float32
    mags = 10.0 ** rng.uniform(-40 if R is np.float32 else -300, 38 if R is np.float32 else 300, 200_000)
    y = (rng.choice([-1.0, 1.0], mags.size) * mags).astype(R)
    y[:100] = 0.0
    for mu, sigma in ((0.0, 1.0), (0.37, 0.77), (-3.0, 1.4999), (1e-3, 3.3e-2)):
        m = H.HmmModel([1.0], [[1.0]], (H.Gaussian(mu, sigma),))
        lb = H.emission_log_matrix(m, y.astype(np.float64) if R is np.float64 else y, dtype=dtype)
        ref = O.emission_matrix([("gaussian", mu, sigma)], y, R)
        got = np.asarray(lb).reshape(-1)
        assert np.array_equal(got, ref[:, 0]), (mu, sigma, int((got != ref[:, 0]).sum()))


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_pipeline_host_slices_match_device_run(dtype):
    """Pipeline.run_from_host (sliced H2D overlapped with the kernels) gives
    the same statistics, log-likelihood and updated model as run() on the
    same observations already on the device."""
    from paper_2605_29208_b200.pipeline import Pipeline

    cfg = make_config("c2", B=96, T=256)
    td = torch.float32 if dtype == "float32" else torch.float64
    y_host = torch.from_numpy(cfg.data).to(td).pin_memory()
    p = Pipeline(cfg.init, cfg.B, cfg.T, dtype)
    p.load(y_host)
    p.run()
    torch.cuda.synchronize()
    ref_tot = p.totals.clone()
    ref_model = p.dm_next.buf.clone()
    ref_path = p.vit.path.clone()
    ref_gamma = p.fb.gamma.clone()
    for slices in (1, 3, 8):
        p.y0.zero_()
        p.run_from_host(y_host, slices=slices)
        torch.cuda.synchronize()
        assert torch.equal(p.totals, ref_tot), slices
        assert torch.equal(p.dm_next.buf, ref_model), slices
        assert torch.equal(p.vit.path, ref_path), slices
        assert torch.equal(p.fb.gamma, ref_gamma), slices


@pytest.mark.parametrize("K", [9, 20, 40, 64])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_large_k_posteriors_xi_and_viterbi(K, dtype):
    """K > 8 (one CTA per sequence, A and the xi accumulators in registers or
    shared memory by size): LL, gamma, log alpha/beta, per-step xi and the
    E-step statistics against the oracle on ragged sequences; Viterbi
    bit-exact."""
    rng = np.random.default_rng(500 + K)
    pi = rng.dirichlet(np.ones(K))
    A = rng.dirichlet(np.ones(K), size=K) * 0.5 + 0.5 * np.eye(K)
    A /= A.sum(1, keepdims=True)
    m = H.HmmModel(pi, A, tuple(H.Poisson(float(r)) for r in np.linspace(0.5, 12.0, K)))
    seqs = [rng.poisson(5.0, n).astype(float) for n in (3, 50, 257)]
    r = H.posteriors_batch(m, seqs, dtype=dtype, include_xi=True)
    lp, la = O.model_tables(pi, A)
    tol = 1e-9 if dtype == "float64" else 1e-5
    X_ = r.xi.cpu().numpy().astype(np.float64)
    for b, y in enumerate(seqs):
        o = O.posteriors(lp, la, O.emission_matrix(to_tuples(m), y), include_xi=True)
        s = slice(r.offsets[b], r.offsets[b + 1])
        xs = slice(r.offsets[b] - b, r.offsets[b + 1] - b - 1)
        assert r.log_likelihood[b].item() == pytest.approx(o["ll"], rel=1e-9 if dtype == "float64" else 1e-4)
        np.testing.assert_allclose(r.gamma[s].double().cpu().numpy(), o["gamma"], atol=tol)
        np.testing.assert_allclose(X_[xs], o["xi"], atol=tol)
    vit = H.viterbi_batch(m, seqs, back=True)
    for b, y in enumerate(seqs):
        p, j, bk = O.viterbi(lp, la, O.emission_matrix(to_tuples(m), y))
        s = slice(vit.offsets[b], vit.offsets[b + 1])
        assert np.array_equal(vit.path[s].cpu().numpy(), p)
        assert np.array_equal(vit.back[s].cpu().numpy().astype(np.int64), bk)
        assert vit.log_joint[b].item() == j
    # E-step statistics (xi totals, gamma totals, Poisson sums) through the fit
    fitted, rep = H.baum_welch(m, seqs, H.TrainingConfig(max_iterations=2, rel_tol=1e-300))
    pi2, A2, em2, trace, _, _ = O.baum_welch(pi, A, to_tuples(m), seqs, 2)
    np.testing.assert_allclose(rep.log_likelihood_trace, trace, rtol=1e-9)
    np.testing.assert_allclose(fitted.transitions, A2, atol=1e-9)


@pytest.mark.parametrize("K", [12, 33])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_large_k_short_sequences_split_pass(K, dtype):
    """Large-K forward-backward on sequences shorter than the T-parallel
    pass's segment count (T = 1, 2, 15, 17: empty and one-step segments) and
    a long one, through the statistics of one Baum-Welch iteration."""
    rng = np.random.default_rng(700 + K)
    pi = rng.dirichlet(np.ones(K))
    A = rng.dirichlet(np.ones(K), size=K) * 0.3 + 0.7 * np.eye(K)
    A /= A.sum(1, keepdims=True)
    m = H.HmmModel(pi, A, tuple(H.Poisson(float(r)) for r in np.linspace(0.5, 9.0, K)))
    seqs = [rng.poisson(4.0, n).astype(float) for n in (1, 2, 15, 17, 400)]
    r = H.posteriors_batch(m, seqs, dtype=dtype, include_xi=True)
    lp, la = O.model_tables(pi, A)
    tol = 1e-9 if dtype == "float64" else 1e-5
    X_ = r.xi.cpu().numpy().astype(np.float64)
    for b, y in enumerate(seqs):
        o = O.posteriors(lp, la, O.emission_matrix(to_tuples(m), y), include_xi=True)
        s = slice(r.offsets[b], r.offsets[b + 1])
        xs = slice(r.offsets[b] - b, r.offsets[b + 1] - b - 1)
        assert r.log_likelihood[b].item() == pytest.approx(o["ll"], rel=1e-9 if dtype == "float64" else 1e-4)
        np.testing.assert_allclose(r.gamma[s].double().cpu().numpy(), o["gamma"], atol=tol)
        np.testing.assert_allclose(r.log_alpha[s].double().cpu().numpy(), o["log_alpha"], rtol=1e-9 if dtype == "float64" else 1e-5, atol=tol)
        np.testing.assert_allclose(r.log_beta[s].double().cpu().numpy(), o["log_beta"], rtol=1e-9 if dtype == "float64" else 1e-5, atol=tol)
        if len(y) > 1:
            np.testing.assert_allclose(X_[xs], o["xi"], atol=tol)
    fitted, rep = H.baum_welch(m, seqs, H.TrainingConfig(max_iterations=2, rel_tol=1e-300), dtype=dtype)
    pi2, A2, em2, trace, _, _ = O.baum_welch(pi, A, to_tuples(m), seqs, 2)
    np.testing.assert_allclose(rep.log_likelihood_trace, trace, rtol=1e-9 if dtype == "float64" else 1e-4)
    np.testing.assert_allclose(fitted.transitions, A2, atol=1e-9 if dtype == "float64" else 1e-4)


@pytest.mark.parametrize("K", [13, 33, 64])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_large_k_viterbi_exact_ties(K, dtype):
    """K > 8 Viterbi with exact candidate ties across the four source lanes of
    a state (uniform A, states sharing a rate): the combined argmax must be
    the reference's first index, path and backpointers bit-exact."""
    rng = np.random.default_rng(900 + K)
    pi = np.full(K, 1.0 / K)
    A = np.full((K, K), 1.0 / K)
    rates = [2.0 + (k % 3) for k in range(K)]  # repeated rates -> tied scores
    m = H.HmmModel(pi, A, tuple(H.Poisson(r) for r in rates))
    seqs = [rng.poisson(3.0, n).astype(float) for n in (1, 40, 300)]
    lp, la = O.model_tables(pi, A)
    vit = H.viterbi_batch(m, seqs, dtype=dtype, back=True)
    for b, y in enumerate(seqs):
        if dtype == "float32":
            lb32 = O.emission_matrix(to_tuples(m), y.astype(np.float32), np.float32)
            p, j, bk = O.viterbi(lp.astype(np.float32), la.astype(np.float32), lb32, np.float32)
        else:
            p, j, bk = O.viterbi(lp, la, O.emission_matrix(to_tuples(m), y))
        s = slice(vit.offsets[b], vit.offsets[b + 1])
        assert np.array_equal(vit.path[s].cpu().numpy(), p)
        assert np.array_equal(vit.back[s].cpu().numpy().astype(np.int64), bk)


def _banded_model(rng, K, half, tie=False, dead_first=False):
    """Banded transitions (structural zeros outside |i - j| <= half), BASELINE
    config 5's shape.  tie: constant band values and repeated rates, so
    candidates tie exactly; dead_first: pi puts all mass on the last state, so
    the low states stay unreachable (-inf scores) for the first steps and some
    columns see only -inf candidates (numpy's argmax then returns index 0)."""
    A = np.zeros((K, K))
    for i in range(K):
        lo, hi = max(0, i - half), min(K, i + half + 1)
        A[i, lo:hi] = 1.0 if tie else rng.dirichlet(np.ones(hi - lo)) * 0.2
        if not tie:
            A[i, i] += 0.8
    A /= A.sum(1, keepdims=True)
    pi = np.zeros(K)
    if dead_first:
        pi[K - 1 if dead_first is True else int(dead_first)] = 1.0
    else:
        pi[:] = 1.0 / K
    rates = [2.0 + (k % 3) for k in range(K)] if tie else list(0.5 * (np.arange(K) + 1))
    return H.HmmModel(pi, A, tuple(H.Poisson(float(r)) for r in rates))


@pytest.mark.parametrize("K", [12, 33, 64])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("variant", ["band", "ties", "dead"])
@pytest.mark.parametrize("sparse", ["1", "0"])
def test_large_k_viterbi_banded_structural_zeros(K, dtype, variant, sparse, monkeypatch):
    _check_banded_viterbi(K, 4, dtype, variant, sparse, monkeypatch)


@pytest.mark.parametrize("half", [2, 5, 6])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_large_k_banded_other_bandwidths(half, dtype, monkeypatch):
    """Band half-widths 2, 5 and 6 (5, 11 and 13 non-zeros per column): the
    5- and 12-entry instantiations of the structural-zero kernels, and a band
    just too wide for them (falls back to the dense kernels)."""
    _check_banded_viterbi(40, half, dtype, "ties", "1", monkeypatch)
    _check_banded_fb(40, half, dtype, "band", "1", monkeypatch)


def _check_banded_viterbi(K, half, dtype, variant, sparse, monkeypatch):
    """K > 8 Viterbi on a banded transition matrix: the structural-zero path
    (finite sources only, an all -inf column mapped to index 0) and the dense
    path give the reference's path, backpointers and log joint bit for bit,
    including exact ties inside the band and columns whose candidates are all
    -inf."""
    monkeypatch.setenv("LOGHMM_VL_SPARSE", sparse)
    rng = np.random.default_rng(1300 + K)
    m = _banded_model(rng, K, half, tie=variant == "ties", dead_first=variant == "dead")
    seqs = [rng.poisson(6.0, n).astype(float) for n in (1, 2, 40, 700)]
    lp, la = O.model_tables(m.initial, m.transitions)
    vit = H.viterbi_batch(m, seqs, dtype=dtype, back=True)
    R = np.float32 if dtype == "float32" else np.float64
    for b, y in enumerate(seqs):
        lb = O.emission_matrix(to_tuples(m), y.astype(R), R)
        with np.errstate(invalid="ignore"):
            p, j, bk = O.viterbi(lp.astype(R), la.astype(R), lb, R)
        s = slice(vit.offsets[b], vit.offsets[b + 1])
        assert np.array_equal(vit.path[s].cpu().numpy(), p), (K, b)
        assert np.array_equal(vit.back[s].cpu().numpy().astype(np.int64), bk), (K, b)
        assert vit.log_joint[b].item() == j


@pytest.mark.parametrize("K", [12, 33, 64])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("variant", ["band", "dead"])
@pytest.mark.parametrize("sparse", ["1", "0"])
def test_large_k_banded_forward_backward(K, dtype, variant, sparse, monkeypatch):
    _check_banded_fb(K, 4, dtype, variant, sparse, monkeypatch)


def _check_banded_fb(K, half, dtype, variant, sparse, monkeypatch):
    """K > 8 forward-backward on a banded transition matrix, through the
    structural-zero sweeps and through the dense ones: LL, log alpha / log
    beta, gamma, per-step xi and one Baum-Welch iteration against the oracle
    (states that are unreachable for the first steps included)."""
    monkeypatch.setenv("LOGHMM_FBL_SPARSE", sparse)
    rng = np.random.default_rng(1700 + K)
    # "dead": all initial mass on one state near the data's rate, so the far
    # states are unreachable (-inf) for the first steps.  (A start that is
    # also wildly inconsistent with the data puts alpha~ and beta~ more than
    # fp32's exponent range apart; that case is exercised in fp64 by the
    # Viterbi test above and documented as an fp32 range limit in DESIGN.md.)
    m = _banded_model(rng, K, half, dead_first=min(K - 1, 11) if variant == "dead" else False)
    seqs = [rng.poisson(6.0, n).astype(float) for n in (1, 2, 17, 40, 700)]
    r = H.posteriors_batch(m, seqs, dtype=dtype, include_xi=True)
    with np.errstate(divide="ignore"):
        lp, la = O.model_tables(m.initial, m.transitions)
    f64 = dtype == "float64"
    tol = 1e-9 if f64 else 1e-5
    X_ = r.xi.cpu().numpy().astype(np.float64)
    for b, y in enumerate(seqs):
        with np.errstate(invalid="ignore", divide="ignore"):
            o = O.posteriors(lp, la, O.emission_matrix(to_tuples(m), y), include_xi=True)
        s = slice(r.offsets[b], r.offsets[b + 1])
        xs = slice(r.offsets[b] - b, r.offsets[b + 1] - b - 1)
        assert r.log_likelihood[b].item() == pytest.approx(o["ll"], rel=1e-9 if f64 else 1e-4)
        np.testing.assert_allclose(r.gamma[s].double().cpu().numpy(), o["gamma"], atol=tol)
        for ours, ref in ((r.log_alpha, o["log_alpha"]), (r.log_beta, o["log_beta"])):
            mine = ours[s].double().cpu().numpy()
            fin = np.isfinite(ref)
            if f64:
                assert np.array_equal(np.isfinite(mine), fin)
            else:
                # the fp32 recursions carry max-normalised linear vectors: entries more
                # than ~87 nats below the step's maximum flush to log 0 = -inf
                assert not np.isfinite(mine[~fin]).any()
                lost = fin & ~np.isfinite(mine)
                rowmax = np.where(fin, ref, -np.inf).max(axis=1, keepdims=True)
                assert (np.broadcast_to(rowmax, ref.shape)[lost] - ref[lost] > 80.0).all()
                # (entries within a few nats of that edge are fp32 denormals: compared loosely)
                fin = fin & np.isfinite(mine) & (rowmax - np.where(fin, ref, -np.inf) < 80.0)
            np.testing.assert_allclose(mine[fin], ref[fin], rtol=1e-9 if f64 else 1e-5, atol=tol if f64 else 2e-4)
        if len(y) > 1:
            np.testing.assert_allclose(X_[xs], o["xi"], atol=tol)
    fitted, rep = H.baum_welch(m, seqs, H.TrainingConfig(max_iterations=2, rel_tol=1e-300), dtype=dtype)
    with np.errstate(invalid="ignore", divide="ignore"):
        pi2, A2, em2, trace, _, _ = O.baum_welch(m.initial, m.transitions, to_tuples(m), seqs, 2)
    np.testing.assert_allclose(rep.log_likelihood_trace, trace, rtol=1e-9 if f64 else 1e-4)
    np.testing.assert_allclose(fitted.transitions, A2, atol=1e-9 if f64 else 1e-4)


def test_large_k_fp32_range_is_reported_not_nan():
    """K > 8 in fp32: a start that is wildly inconsistent with the data puts
    the max-normalised forward and backward vectors further apart than fp32's
    exponent range.  The reference (fp64 log space) and the fp64 path return
    finite posteriors; the fp32 path must say so instead of returning NaN."""
    rng = np.random.default_rng(1764)
    m = _banded_model(rng, 64, 4, dead_first=True)  # all initial mass on the rate-32 state
    seqs = [rng.poisson(6.0, n).astype(float) for n in (17, 700)]
    r64 = H.posteriors_batch(m, seqs, dtype="float64")
    assert torch.isfinite(r64.gamma).all()
    with pytest.raises(FloatingPointError, match="float64"):
        H.posteriors_batch(m, seqs, dtype="float32")
    with pytest.raises(FloatingPointError, match="float64"):
        H.baum_welch(m, seqs, H.TrainingConfig(max_iterations=2), dtype="float32")


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_error_semantics_equal_length_batches(dtype):
    """Error paths of the equal-length decomposition (chunk operators + meet in
    the middle for fp32): a dead observation, an unreachable path and NaN are
    reported with the reference's exceptions, sequence and index."""
    rng = np.random.default_rng(3)
    m = H.HmmModel([0.5, 0.5], [[0.9, 0.1], [0.2, 0.8]], (H.Poisson(2.0), H.Poisson(5.0)))
    data = rng.poisson(3.0, size=(4, 64)).astype(np.float64)
    dead = data.copy()
    dead[2, 37] = 0.5  # outside the support of every state
    with pytest.raises(H.InfeasibleSequenceError, match="sequence impossible under model"):
        H.posteriors_batch(m, dead, dtype=dtype)
    with pytest.raises(H.TrainingError, match="sequence 2, index 37"):
        H.baum_welch(m, [dead[b] for b in range(4)], H.TrainingConfig(max_iterations=2))
    nan = data.copy()
    nan[1, 50] = np.nan
    with pytest.raises(ValueError, match="NaN"):
        H.posteriors_batch(m, nan, dtype=dtype)
    # impossible without a dead row: state 1 (Gaussian) is unreachable, and
    # y <= 0 is outside the support of state 0 (Gamma) only
    m2 = H.HmmModel([1.0, 0.0], [[1.0, 0.0], [0.0, 1.0]], (H.Gamma(2.0, 1.0), H.Gaussian(0.0, 1.0)))
    ok = rng.gamma(2.0, 1.0, size=(4, 64))
    bad = ok.copy()
    bad[3, 10] = -1.0
    r = H.posteriors_batch(m2, bad, dtype=dtype, check=False)
    ll = r.log_likelihood.cpu().numpy()
    assert np.isfinite(ll[:3]).all() and ll[3] == -np.inf
    with pytest.raises(H.InfeasibleSequenceError, match="sequence impossible under model"):
        H.posteriors_batch(m2, bad, dtype=dtype)
    with pytest.raises(H.TrainingError, match="sequence 3 is impossible"):
        H.baum_welch(m2, [bad[b] for b in range(4)], H.TrainingConfig(max_iterations=2))
