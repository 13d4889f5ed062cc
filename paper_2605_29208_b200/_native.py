"""ctypes binding of the C ABI in include/loghmm_b200.h.

This is the only place the package touches native code.  The library is built
in-tree (paper_2605_29208_b200/_lib/libloghmm_b200.so, see csrc/Makefile) and
loaded on first use; if it is missing every compute entry point raises
``NativeLibraryError`` -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

__all__ = [
    "NativeLibraryError",
    "lib",
    "library_path",
    "MODEL_DTYPE",
    "EMISSION_DTYPE",
    "MAX_STATES",
    "NSLOT",
    "FAM",
    "F32",
    "F64",
    "GUARD_CANDIDATES",
    "EXPORTED_SYMBOLS",
    "check",
]

MAX_STATES = 64
MAX_STREAMS = 2
NSLOT = 6
GUARD_CANDIDATES = 8
F32, F64 = 0, 1
FAM = {"none": 0, "gaussian": 1, "student_t": 2, "gamma": 3, "von_mises": 4, "poisson": 5,
       "lognormal": 6, "exponential": 7, "rayleigh": 8, "uniform": 9, "categorical": 10, "beta": 11,
       "weibull": 12, "negative_binomial": 13, "chi_squared": 14, "pareto": 15}
EXT_FAMILIES = frozenset(n for n, v in FAM.items() if v >= 6)  # fitted by csrc/hmm_extfit.cuh

# Mirrors loghmm_emission_t / loghmm_model_t (natural alignment, no padding).
EMISSION_DTYPE = np.dtype(
    [("family", "<i4"), ("reserved", "<i4"), ("p", "<f8", (4,)), ("c", "<f8", (4,))]
)
MODEL_DTYPE = np.dtype(
    [
        ("K", "<i4"),
        ("n_streams", "<i4"),
        ("reserved", "<i4", (2,)),
        ("em", EMISSION_DTYPE, (MAX_STREAMS, MAX_STATES)),
        ("pi", "<f8", (MAX_STATES,)),
        ("A", "<f8", (MAX_STATES * MAX_STATES,)),
        ("log_pi", "<f8", (MAX_STATES,)),
        ("log_A", "<f8", (MAX_STATES * MAX_STATES,)),
    ]
)

# status codes (loghmm_mstep_status)
MS_UPDATED = 0
MS_COLLAPSED = 1
MS_ERR_NO_MASS = 16
MS_ERR_SUPPORT = 17
MS_ERR_GAMMA_VAR = 18
MS_ERR_GAMMA_GAP = 19
MS_ERR_NONFINITE = 20
MS_ERR_DEGENERATE = 21
MS_ERR_CAT_CODE = 22
MS_WARN_NEWTON = 1 << 8
MS_WARN_CEILING = 1 << 9
MS_WARN_BOUNDARY = 1 << 10
MS_WARN_ITERCAP = 1 << 11
MS_STUDENT_GUARD = 1 << 12
MS_EXT_FIT = 1 << 13
EXT_MAX_PASSES = 64
BIN_SLOTS = 22

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double
_sz = ctypes.c_size_t

# name -> (restype, argtypes); every symbol declared in include/loghmm_b200.h
_SIGNATURES = {
    "loghmm_abi_version": (_i32, []),
    "loghmm_model_bytes": (_sz, []),
    "loghmm_stats_width": (_i64, [_i32, _i32]),
    "loghmm_fb_workspace_bytes": (_sz, [_i32, _i32, _i64, _i64, _i64]),
    "loghmm_viterbi_workspace_bytes": (_sz, [_i32, _i32, _i64, _i64, _i64]),
    "loghmm_emission": (_i32, [_i32, _vp, _vp, _vp, _vp, _i64, _vp, _i32, _vp, _vp]),
    "loghmm_forward_backward": (
        _i32,
        [_i32, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _vp, _vp, _vp,
         _vp, _vp, _vp, _sz, _vp],
    ),
    "loghmm_viterbi": (
        _i32,
        [_i32, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _vp, _vp, _vp,
         _sz, _vp],
    ),
    "loghmm_reduce_stats": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "loghmm_mstep": (_i32, [_vp, _vp, _i64, _f64, _f64, _f64, _i32, _f64, _vp, _vp, _vp, _vp]),
    "loghmm_reduce_workspace_bytes": (_sz, [_i64, _i64]),
    "loghmm_reduce_mstep": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp, _i64, _f64, _f64, _f64, _i32,
                                   _f64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "loghmm_variance_pass": (_i32, [_i32, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "loghmm_guard_workspace_bytes": (_sz, [_i32, _i64]),
    "loghmm_student_guard": (
        _i32,
        [_i32, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp],
    ),
    "loghmm_bin_moments": (_i32, [_vp, _i64, _i32, _vp, _vp]),
    "loghmm_ext_fit_pass": (_i32, [_i32, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "loghmm_variance_partial": (_i32, [_i32, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "loghmm_variance_finish": (_i32, [_vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "loghmm_student_guard_partial": (
        _i32, [_i32, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "loghmm_student_guard_select": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
}
EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_STATUS = {
    0: "ok",
    1: "invalid argument",
    2: "unsupported shape/family",
    3: "CUDA launch error",
    4: "workspace too small",
}


class NativeLibraryError(RuntimeError):
    """The sm_100a extension is missing or failed; there is no fallback."""


def library_path() -> Path:
    env = os.environ.get("LOGHMM_B200_LIB")
    if env:
        return Path(env)
    return Path(__file__).resolve().parent / "_lib" / "libloghmm_b200.so"


_LIB = None


def lib():
    """Load (once) and return the native library with typed signatures."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = library_path()
    if not path.exists():
        raise NativeLibraryError(
            f"native library not built: {path} (run `make -C paper_2605_29208_b200/csrc` "
            "or __graft_entry__.build()); the CUDA path has no CPU fallback"
        )
    try:
        handle = ctypes.CDLL(str(path))
    except OSError as exc:  # pragma: no cover - environment specific
        raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
    # an explicit LOGHMM_B200_LIB override (A/B runs against an older build)
    # may lack entry points added since; the in-tree library must have all
    override = bool(os.environ.get("LOGHMM_B200_LIB"))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(handle, name, None) if override else getattr(handle, name)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    if handle.loghmm_model_bytes() != MODEL_DTYPE.itemsize:
        raise NativeLibraryError(
            f"loghmm_model_t size mismatch: C {handle.loghmm_model_bytes()} vs "
            f"numpy {MODEL_DTYPE.itemsize}"
        )
    _LIB = handle
    return handle


def check(code: int, what: str) -> None:
    if code != 0:
        raise NativeLibraryError(f"{what} failed: {_STATUS.get(code, code)}")
