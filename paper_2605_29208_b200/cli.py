"""``loghmm`` command line (fit / decode / eval / benchmark, the reference's
cli.py:141-257) with the hot path on the B200 core.

    python -m paper_2605_29208_b200.cli decode --model m.json --data obs.csv

The reference's own CLI module (argument parsing, file formats, output
formatting, exit codes) runs unchanged; ``compat.install`` rebinds the
functions it calls -- posteriors, viterbi, baum_welch, score_model,
default_initial_model, read_sequences -- to the drop-in, so the numbers come
from the device kernels.  Needs the reference package importable (``loghmm``,
e.g. the baseline/_ref install).
"""

from __future__ import annotations

import sys
from pathlib import Path

_REF_INSTALL = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


def main(argv=None) -> int:
    try:
        import loghmm  # noqa: F401
    except ImportError:
        if (_REF_INSTALL / "loghmm").exists():
            sys.path.insert(0, str(_REF_INSTALL))
        import loghmm  # noqa: F401
    import loghmm.cli

    from . import compat

    handle = compat.install(loghmm)
    try:
        return loghmm.cli.main(argv)
    finally:
        handle.uninstall()


if __name__ == "__main__":
    raise SystemExit(main())
