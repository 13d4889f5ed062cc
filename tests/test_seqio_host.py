"""Host-side parity of the sequence reader (paper_2605_29208_b200.seqio)
with the reference's read_sequences (model_io.py:150-195): same sequences,
same error texts.  Uses the unmodified reference (baseline/_ref install or
/root/reference) where present."""

import io
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2605_29208_b200 import seqio

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def ref_read():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "loghmm").exists():
            sys.path.insert(0, str(p))
            from loghmm.model_io import read_sequences

            return read_sequences
    pytest.skip("reference package not available")


TEXTS = [
    "y\n1.0\n2.5\n\n3\n4\n5\n",
    "a,b\n1,2\n3,4\n\n\n5,6\n",
    "1\n2\n3",
    "time;value\n0;1.5\n1;-2.25e-3\n\n2;7\n",
    "  1.0  \n\t2.0\n\n\n\n3.0\n\n",
    "1\r\n2\r\n\r\n3\r\n",
    "1\x0c2\n\n3\n",
]
BAD = ["1\n2\nx\n", "1,2\n3\n", "1\nnan\n", "\n\n", "header\nother\n"]


@pytest.mark.parametrize("k", range(len(TEXTS)))
def test_same_sequences(ref_read, k):
    text = TEXTS[k]
    col = 1 if "," in text or ";" in text else 0
    delim = ";" if ";" in text else ","
    ref = ref_read(io.StringIO(text), column=col, delimiter=delim)
    got = seqio.read_sequences(io.StringIO(text), column=col, delimiter=delim)
    assert len(ref) == len(got)
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("k", range(len(BAD)))
def test_same_errors(ref_read, k):
    text = BAD[k]
    with pytest.raises(ValueError) as e1:
        ref_read(io.StringIO(text), column=1 if text.startswith("1,2") else 0)
    with pytest.raises(ValueError) as e2:
        seqio.read_sequences(io.StringIO(text), column=1 if text.startswith("1,2") else 0)
    assert str(e1.value) == str(e2.value)


def test_file_path(ref_read, tmp_path):
    p = tmp_path / "obs.csv"
    p.write_text("v\n" + "\n".join(str(x) for x in range(100)) + "\n\n" + "\n".join("1.5" for _ in range(7)))
    ref = ref_read(p)
    got = seqio.read_sequences(p)
    assert [a.tolist() for a in ref] == [b.tolist() for b in got]
    with pytest.raises(OSError, match="could not read sequences"):
        seqio.read_sequences(tmp_path / "missing.csv")
