"""default_initial_model on the device (device sort + loghmm_bin_moments)
against the unmodified reference's default_initial_model (training.py:
239-282) for every family, where the reference install (baseline/_ref) is
present, and against the np.array_split rule restated here otherwise.
Seeds agree to 1e-12 relative (the bin sums are reduced in a different
order than numpy's dot)."""

import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2605_29208_b200 as H  # noqa: E402

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_array_split_rule():
    y = np.array([3.0, 1.0, 2.0, 10.0, 12.0, 11.0, 0.0])
    m = H.default_initial_model(2, "poisson", [y])
    bins = np.array_split(np.sort(y), 2)
    assert [d.rate for d in m.emissions] == pytest.approx([float(np.mean(b)) for b in bins], rel=1e-15)
    assert np.allclose(m.transitions, [[0.9, 0.1], [0.1, 0.9]])
    with pytest.raises(H.TrainingError, match="more states than observations"):
        H.default_initial_model(5, "gaussian", [np.array([1.0, 2.0])])
    with pytest.raises(ValueError, match="expected 1 or 3 family names"):
        H.default_initial_model(3, ["gaussian", "poisson"], [y])


DATA = {
    "gaussian": lambda r: r.normal(0, 2, 500),
    "lognormal": lambda r: r.lognormal(0, 1, 500),
    "exponential": lambda r: r.exponential(2.0, 500),
    "poisson": lambda r: r.poisson(4.0, 500).astype(float),
    "rayleigh": lambda r: r.rayleigh(1.5, 500),
    "uniform": lambda r: r.uniform(-1, 3, 500),
    "categorical": lambda r: r.integers(0, 4, 500).astype(float),
    "von_mises": lambda r: r.vonmises(0.5, 2.0, 500),
    "gamma": lambda r: r.gamma(2.0, 1.5, 500),
    "beta": lambda r: r.beta(2.0, 3.0, 500),
    "weibull": lambda r: 2.0 * r.weibull(1.5, 500),
    "negative_binomial": lambda r: r.negative_binomial(3, 0.4, 500).astype(float),
    "chi_squared": lambda r: r.chisquare(4.0, 500),
    "pareto": lambda r: 1.0 + r.pareto(2.0, 500),
    "student_t": lambda r: r.standard_t(5, 500),
}


@pytest.mark.parametrize("fam", sorted(DATA))
def test_matches_reference_default_initial_model(fam):
    if not (REF / "loghmm").exists():
        pytest.skip("reference install baseline/_ref absent")
    sys.path.insert(0, str(REF))
    from loghmm.training import default_initial_model as ref_init

    rng = np.random.default_rng(hash(fam) % 1000)
    seqs = [DATA[fam](rng)[:n] for n in (500, 321)]
    ref = ref_init(3, fam, seqs)
    got = H.default_initial_model(3, fam, seqs)
    np.testing.assert_allclose(got.initial, ref.initial, rtol=0)
    np.testing.assert_allclose(got.transitions, ref.transitions, rtol=0)
    for a, b in zip(got.emissions, ref.emissions):
        assert a.family == b.family
        np.testing.assert_allclose(list(a.params().values()), list(b.params().values()), rtol=1e-12, atol=1e-15)


def test_support_errors_match_reference():
    with pytest.raises(ValueError, match="gamma fit requires strictly positive observations"):
        H.default_initial_model(2, "gamma", [np.array([1.0, -2.0, 3.0, 4.0])])
    with pytest.raises(ValueError, match="beta fit requires observations strictly inside"):
        H.default_initial_model(2, "beta", [np.array([0.5, 0.2, 1.0, 0.3])])
