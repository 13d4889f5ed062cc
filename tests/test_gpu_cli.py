"""The reference's command line on the B200 core (paper_2605_29208_b200.cli:
the unmodified loghmm CLI with the hot path rebound by compat.install), run
against the same CLI on the CPU.  decode text output must be byte-identical
(integer states); eval / fit numbers agree to 1e-9 relative.  Needs the
reference install baseline/_ref (skipped where absent)."""

import io
import json
import sys
from contextlib import redirect_stdout
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module")
def files(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not (REF / "loghmm").exists():
        pytest.skip("reference install baseline/_ref absent")
    sys.path.insert(0, str(REF))
    import loghmm
    from loghmm.model_io import save_model

    d = tmp_path_factory.mktemp("cli")
    rng = np.random.default_rng(3)
    model = loghmm.HmmModel([0.5, 0.5], [[0.9, 0.1], [0.2, 0.8]],
                            (loghmm.Gaussian(-1.0, 0.8), loghmm.Gaussian(2.0, 1.1)))
    save_model(model, d / "model.json")
    lines = ["value"]
    for n in (200, 150, 90):
        s, st = [], 0
        for _ in range(n):
            s.append(rng.normal(-1.0, 0.8) if st == 0 else rng.normal(2.0, 1.1))
            st = st if rng.random() < 0.9 else 1 - st
        lines += [repr(v) for v in s] + [""]
    (d / "obs.csv").write_text("\n".join(lines) + "\n")
    return d


def run(argv, gpu):
    import loghmm.cli

    from paper_2605_29208_b200 import cli

    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = cli.main(argv) if gpu else loghmm.cli.main(argv)
    return rc, buf.getvalue()


def test_decode_byte_identical(files):
    for method in ("viterbi", "posterior"):
        argv = ["decode", "--model", str(files / "model.json"), "--data", str(files / "obs.csv"),
                "--method", method]
        rc_c, out_c = run(argv, gpu=False)
        rc_g, out_g = run(argv, gpu=True)
        assert rc_c == rc_g == 0
        assert out_g == out_c


def test_eval_and_fit_numbers(files):
    argv = ["eval", "--model", str(files / "model.json"), "--data", str(files / "obs.csv"), "--format", "json"]
    c = json.loads(run(argv, gpu=False)[1])
    g = json.loads(run(argv, gpu=True)[1])
    assert c.keys() == g.keys()
    for k in c:
        if isinstance(c[k], float):
            assert g[k] == pytest.approx(c[k], rel=1e-9), k
        else:
            assert g[k] == c[k], k
    argv = ["fit", "--data", str(files / "obs.csv"), "--states", "2", "--family", "gaussian",
            "--format", "json", "--max-iter", "30"]
    rc_c, out_c = run(argv, gpu=False)
    rc_g, out_g = run(argv, gpu=True)
    assert rc_c == rc_g
    c, g = json.loads(out_c), json.loads(out_g)
    assert g["iterations"] == c["iterations"] and g["converged"] == c["converged"]
    assert g["log_likelihood"] == pytest.approx(c["log_likelihood"], rel=1e-9)


def test_benchmark_runs(files):
    rc, out = run(["benchmark", "--lengths", "100,1000"], gpu=True)
    assert rc == 0 and out.splitlines()[0] == "length,forward_backward_ms,obs_per_ms"
