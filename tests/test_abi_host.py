"""CPU-side checks: the C-ABI library loads and exports every symbol the
header declares; host-side model encoding, validation and error texts."""

import math
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2605_29208_b200 import _native
from paper_2605_29208_b200.distributions import Gamma, Gaussian, Joint, Poisson, StudentT, VonMises
from paper_2605_29208_b200.engine import encode_model
from paper_2605_29208_b200.inference import HmmModel
from paper_2605_29208_b200.training import TrainingConfig

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "loghmm_b200.h").read_text()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(loghmm_\w+)\(", text, flags=re.M)))


def test_header_declares_bound_symbols():
    assert sorted(_native.EXPORTED_SYMBOLS) == header_symbols()


def test_library_loads_and_exports():
    lib = _native.lib()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.loghmm_abi_version() == 1
    assert lib.loghmm_model_bytes() == _native.MODEL_DTYPE.itemsize
    assert lib.loghmm_stats_width(4, 1) == 16 + 8 + 2 * 4 * 6


def test_model_validation_messages():
    with pytest.raises(ValueError, match="transitions"):
        HmmModel([1.0], [[0.8]], (Gaussian(0, 1),))
    with pytest.raises(ValueError, match="initial"):
        HmmModel([0.5, 0.4], [[0.5, 0.5], [0.5, 0.5]], (Gaussian(0, 1), Gaussian(1, 1)))
    with pytest.raises(ValueError, match="emission"):
        HmmModel([0.5, 0.5], [[0.5, 0.5], [0.5, 0.5]], (Gaussian(0, 1),))
    with pytest.raises(ValueError, match="sigma"):
        Gaussian(0.0, 0.0)
    with pytest.raises(ValueError, match=r"von_mises.mu must lie in \(-pi, pi\]"):
        VonMises(-math.pi, 1.0)
    with pytest.raises(ValueError):
        TrainingConfig(rel_tol=0.0)


def test_encode_model_constants_match_reference_math():
    m = HmmModel([0.25, 0.75], [[0.9, 0.1], [0.0, 1.0]],
                 (Gaussian(0.5, 2.0), StudentT(0.1, 0.3, 4.5)))
    rec = encode_model(m)
    assert rec["K"] == 2 and rec["n_streams"] == 1
    g = rec["em"][0, 0]
    assert g["family"] == _native.FAM["gaussian"]
    assert g["c"][0] == -0.5 * math.log(2.0 * math.pi) - math.log(2.0)
    s = rec["em"][0, 1]
    nu = 4.5
    assert s["c"][0] == (math.lgamma((nu + 1) / 2) - math.lgamma(nu / 2)
                         - 0.5 * math.log(nu * math.pi) - math.log(0.3))
    assert rec["log_A"][3] == 0.0 and rec["log_A"][2] == -np.inf
    assert np.array_equal(rec["log_pi"][:2], np.log([0.25, 0.75]))


def test_encode_joint_model():
    m = HmmModel([1.0], [[1.0]], (Joint(Gamma(2.0, 3.0), VonMises(0.5, 2.0)),))
    rec = encode_model(m)
    assert rec["n_streams"] == 2
    assert rec["em"][0, 0]["family"] == _native.FAM["gamma"]
    assert rec["em"][1, 0]["family"] == _native.FAM["von_mises"]
    assert rec["em"][0, 0]["c"][1] == 1.0


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_29208_b200 import NativeLibraryError, posteriors

    with pytest.raises(NativeLibraryError):
        posteriors(HmmModel([1.0], [[1.0]], (Poisson(2.0),)), np.array([1.0, 2.0]))
