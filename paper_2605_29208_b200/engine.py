"""Device-side plumbing: batch packing, model blocks, workspaces, launches.

PyTorch owns every device buffer (allocation, streams); the arithmetic is in
the sm_100a kernels behind the C ABI (_native).  Nothing here computes on the
CPU beyond packing inputs and reading back small flag / statistic arrays.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._native import F32, F64, MODEL_DTYPE, check, lib

__all__ = [
    "Batch",
    "DeviceModel",
    "make_batch",
    "encode_model",
    "forward_backward",
    "viterbi",
    "emission",
    "reduce_stats",
    "mstep",
    "student_guard",
    "torch_dtype",
    "LUT_SIZE",
]

LUT_SIZE = 4096
_LUTS: dict = {}


def torch_dtype(dtype) -> torch.dtype:
    if dtype in ("float32", "fp32", "f32", np.float32, torch.float32):
        return torch.float32
    if dtype in ("float64", "fp64", "f64", float, np.float64, torch.float64, None):
        return torch.float64
    raise ValueError(f"unsupported dtype {dtype!r}; use float32 or float64")


def _code(td: torch.dtype) -> int:
    return F32 if td == torch.float32 else F64


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise _native.NativeLibraryError(
            "no CUDA device: the loghmm B200 core runs on the GPU only (no CPU fallback)"
        )
    return torch.device("cuda", torch.cuda.current_device())


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def lgamma_lut(device) -> torch.Tensor:
    """Host table of math.lgamma(n + 1.0) (the reference's Poisson term,
    distributions.py:80-86, 259) uploaded once per device."""
    key = str(device)
    if key not in _LUTS:
        host = np.array([math.lgamma(n + 1.0) for n in range(LUT_SIZE)], dtype=np.float64)
        _LUTS[key] = torch.from_numpy(host).to(device)
    return _LUTS[key]


# ---------------------------------------------------------------------------
# batches
# ---------------------------------------------------------------------------
@dataclass
class Batch:
    """Sequences packed back to back (training.py:172 layout)."""

    y0: torch.Tensor  # [N]
    y1: torch.Tensor | None  # [N] second stream (joint emissions)
    offsets: torch.Tensor  # [B+1] int64, device
    offsets_host: np.ndarray  # [B+1] int64
    dtype: torch.dtype

    @property
    def B(self) -> int:
        return len(self.offsets_host) - 1

    @property
    def N(self) -> int:
        return int(self.offsets_host[-1])

    @property
    def max_T(self) -> int:
        return int(np.max(np.diff(self.offsets_host))) if self.B else 0

    @property
    def lengths(self) -> np.ndarray:
        return np.diff(self.offsets_host)


_SEQ_ERR = "an observation sequence must be a non-empty 1-D array"


def make_batch(data, n_streams: int = 1, dtype="float64", device=None) -> Batch:
    """Pack observations into a device Batch.

    Accepts a 1-D sequence, a [B, T] array/tensor, or a list of 1-D sequences
    (ragged allowed); for two-stream models each sequence is [T, 2] and a
    batch is [B, T, 2].
    """
    td = torch_dtype(dtype)
    dev = device or _device()
    if isinstance(data, Batch):
        return data
    if torch.is_tensor(data) or isinstance(data, np.ndarray):
        arr = data
        nd = arr.ndim
        if nd == n_streams:  # single sequence
            arr = arr[None]
            nd += 1
        if nd != n_streams + 1:
            raise ValueError(_SEQ_ERR)
        B, T = int(arr.shape[0]), int(arr.shape[1])
        if T < 1 or B < 1:
            raise ValueError(_SEQ_ERR)
        if isinstance(arr, np.ndarray):
            arr = np.ascontiguousarray(arr)  # (reversed / strided views)
        t = torch.as_tensor(arr)
        t = t.to(device=dev, dtype=td, non_blocking=True)
        if n_streams == 1:
            y0, y1 = t.reshape(-1).contiguous(), None
        else:
            if t.shape[-1] != 2:
                raise ValueError("joint observations must have a trailing dimension of 2")
            y0 = t[..., 0].reshape(-1).contiguous()
            y1 = t[..., 1].reshape(-1).contiguous()
        off = np.arange(B + 1, dtype=np.int64) * T
    else:
        seqs = list(data)
        if not seqs:
            raise ValueError("training data contains no sequences")
        host = []
        for s in seqs:
            a = s.detach().cpu().numpy() if torch.is_tensor(s) else np.asarray(s, dtype=np.float64)
            if a.ndim != n_streams or a.shape[0] < 1:
                raise ValueError(_SEQ_ERR)
            host.append(np.asarray(a, dtype=np.float64))
        lens = np.array([h.shape[0] for h in host], dtype=np.int64)
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        cat = np.concatenate(host, axis=0)
        t = torch.from_numpy(cat).to(device=dev, dtype=td)
        if n_streams == 1:
            y0, y1 = t.contiguous(), None
        else:
            y0, y1 = t[:, 0].contiguous(), t[:, 1].contiguous()
    offsets = torch.from_numpy(off).to(dev)
    return Batch(y0=y0, y1=y1, offsets=offsets, offsets_host=off, dtype=td)


# ---------------------------------------------------------------------------
# model blocks
# ---------------------------------------------------------------------------
def encode_model(model) -> np.ndarray:
    """loghmm_model_t for an HmmModel; log pi / log A are the reference's own
    np.log values (inference.py:82-88)."""
    rec = np.zeros((), dtype=MODEL_DTYPE)
    K = model.num_states
    if K > _native.MAX_STATES:
        raise ValueError(f"at most {_native.MAX_STATES} states are supported, got {K}")
    ems = model.emissions
    n_streams = ems[0].n_streams
    if any(e.n_streams != n_streams for e in ems):
        raise ValueError("all states must use the same number of observation streams")
    rec["K"] = K
    rec["n_streams"] = n_streams
    for j, e in enumerate(ems):
        parts = (e.first, e.second) if n_streams == 2 else (e,)
        for s, d in enumerate(parts):
            r = d.record()
            fam, p, c = r[:3]
            rec["em"][s, j]["reserved"] = r[3] if len(r) > 3 else 0  # categorical: category count
            rec["em"][s, j]["family"] = fam
            rec["em"][s, j]["p"] = p
            rec["em"][s, j]["c"] = c
    rec["pi"][:K] = model.initial
    rec["A"][: K * K] = np.asarray(model.transitions).reshape(-1)
    rec["log_pi"][:K] = model.log_initial()
    rec["log_A"][: K * K] = model.log_transitions().reshape(-1)
    return rec


class DeviceModel:
    """A loghmm_model_t living in device memory plus its host descriptor."""

    def __init__(self, host_record: np.ndarray, device):
        self.host = np.array(host_record, dtype=MODEL_DTYPE)  # own copy (descriptor)
        raw = np.frombuffer(self.host.tobytes(), dtype=np.uint8)
        self.buf = torch.from_numpy(raw.copy()).to(device)

    @classmethod
    def from_model(cls, model, device=None):
        return cls(encode_model(model), device or _device())

    @classmethod
    def empty_like(cls, other: "DeviceModel"):
        obj = cls.__new__(cls)
        obj.host = np.array(other.host, dtype=MODEL_DTYPE)
        obj.buf = torch.empty_like(other.buf)
        return obj

    @property
    def K(self) -> int:
        return int(self.host["K"])

    @property
    def n_streams(self) -> int:
        return int(self.host["n_streams"])

    def desc_ptr(self) -> int:
        return self.host.ctypes.data

    def ptr(self) -> int:
        return int(self.buf.data_ptr())

    def to_host(self) -> np.ndarray:
        raw = self.buf.cpu().numpy()
        return np.frombuffer(raw.tobytes(), dtype=MODEL_DTYPE)[0]


# ---------------------------------------------------------------------------
# launches
# ---------------------------------------------------------------------------
def emission(batch: Batch, dm: DeviceModel) -> torch.Tensor:
    L = lib()
    out = torch.empty((batch.N, dm.K), dtype=batch.dtype, device=batch.y0.device)
    lut = lgamma_lut(batch.y0.device)
    check(
        L.loghmm_emission(_code(batch.dtype), dm.desc_ptr(), dm.ptr(), _ptr(batch.y0),
                          _ptr(batch.y1), batch.N, _ptr(lut), LUT_SIZE, _ptr(out), _stream()),
        "loghmm_emission",
    )
    return out


@dataclass
class FBOutputs:
    log_alpha: torch.Tensor | None
    log_beta: torch.Tensor | None
    gamma: torch.Tensor | None
    xi: torch.Tensor | None
    ll: torch.Tensor
    partials: torch.Tensor | None
    flags: torch.Tensor


class Workspace:
    """Grow-only device scratch owned by the caller (the library allocates nothing)."""

    def __init__(self):
        self._buf = None

    def get(self, nbytes: int, device) -> tuple[int, int]:
        if nbytes == 0:
            return 0, 0
        if self._buf is None or self._buf.numel() < nbytes or self._buf.device != device:
            # zero-filled once: the reduction / variance passes keep their
            # inter-block counters here and leave them at zero
            self._buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        return int(self._buf.data_ptr()), int(self._buf.numel())


_WS_FB = Workspace()
_WS_VIT = Workspace()
_WS_GUARD = Workspace()


def forward_backward(batch: Batch, dm: DeviceModel, *, alpha=True, beta=True, gamma=True,
                     xi=False, stats=False, out: FBOutputs | None = None,
                     workspace: Workspace | None = None) -> FBOutputs:
    L = lib()
    dev = batch.y0.device
    K, B, N = dm.K, batch.B, batch.N
    td = batch.dtype
    if out is None:
        width = int(L.loghmm_stats_width(K, dm.n_streams))
        out = FBOutputs(
            log_alpha=torch.empty((N, K), dtype=td, device=dev) if alpha else None,
            log_beta=torch.empty((N, K), dtype=td, device=dev) if beta else None,
            gamma=torch.empty((N, K), dtype=td, device=dev) if gamma else None,
            xi=torch.empty((max(N - B, 0), K, K), dtype=td, device=dev) if xi else None,
            ll=torch.empty(B, dtype=torch.float64, device=dev),
            partials=torch.empty((B, width), dtype=torch.float64, device=dev) if stats else None,
            flags=torch.empty((B, 2), dtype=torch.int64, device=dev),
        )
    code = _code(td)
    ws = workspace or _WS_FB
    need = int(L.loghmm_fb_workspace_bytes(code, K, B, N, batch.max_T))
    wptr, wlen = ws.get(need, dev)
    lut = lgamma_lut(dev)
    check(
        L.loghmm_forward_backward(
            code, dm.desc_ptr(), dm.ptr(), _ptr(batch.y0), _ptr(batch.y1), _ptr(batch.offsets),
            B, N, batch.max_T, _ptr(lut), LUT_SIZE, _ptr(out.log_alpha), _ptr(out.log_beta),
            _ptr(out.gamma), _ptr(out.xi), _ptr(out.ll), _ptr(out.partials), _ptr(out.flags),
            wptr, wlen, _stream(),
        ),
        "loghmm_forward_backward",
    )
    return out


@dataclass
class VitOutputs:
    path: torch.Tensor
    log_joint: torch.Tensor
    back: torch.Tensor | None
    flags: torch.Tensor


def viterbi(batch: Batch, dm: DeviceModel, *, back=False, out: VitOutputs | None = None,
            workspace: Workspace | None = None) -> VitOutputs:
    L = lib()
    dev = batch.y0.device
    K, B, N = dm.K, batch.B, batch.N
    if out is None:
        out = VitOutputs(
            path=torch.empty(N, dtype=torch.int64, device=dev),
            log_joint=torch.empty(B, dtype=torch.float64, device=dev),
            back=torch.empty((N, K), dtype=torch.uint8, device=dev) if back else None,
            flags=torch.zeros((B, 2), dtype=torch.int64, device=dev),
        )
    code = _code(batch.dtype)
    ws = workspace or _WS_VIT
    need = int(L.loghmm_viterbi_workspace_bytes(code, K, B, N, batch.max_T))
    wptr, wlen = ws.get(need, dev)
    lut = lgamma_lut(dev)
    check(
        L.loghmm_viterbi(
            code, dm.desc_ptr(), dm.ptr(), _ptr(batch.y0), _ptr(batch.y1), _ptr(batch.offsets),
            B, N, batch.max_T, _ptr(lut), LUT_SIZE, _ptr(out.path), _ptr(out.log_joint),
            _ptr(out.back), _ptr(out.flags), wptr, wlen, _stream(),
        ),
        "loghmm_viterbi",
    )
    return out


def reduce_stats(partials: torch.Tensor, ll: torch.Tensor, out: torch.Tensor | None = None):
    L = lib()
    B, width = partials.shape
    if out is None:
        out = torch.empty(width + 1, dtype=torch.float64, device=partials.device)
    check(L.loghmm_reduce_stats(_ptr(partials), _ptr(ll), B, width, _ptr(out), _stream()),
          "loghmm_reduce_stats")
    return out


_WS_RED = Workspace()


def reduce_mstep(partials: torch.Tensor, ll: torch.Tensor, totals: torch.Tensor,
                 dm_in: DeviceModel | None = None, n_sequences: int = 0, config=None,
                 dm_out: DeviceModel | None = None, status: torch.Tensor | None = None,
                 guard: torch.Tensor | None = None, td: torch.dtype = torch.float64,
                 workspace: Workspace | None = None) -> torch.Tensor:
    """Fused single-rank reduction + M-step (reduction only when dm_in is None)."""
    L = lib()
    B, width = partials.shape
    ws = workspace if workspace is not None else _WS_RED
    wptr, wlen = ws.get(int(L.loghmm_reduce_workspace_bytes(B, width)), partials.device)
    if dm_in is None:
        args = (None, 0, 0.0, 0.0, 0.0, 0, 0.0, None, None, None)
    else:
        e = config.ecme
        args = (dm_in.ptr(), n_sequences, float(config.collapse_epsilon), float(e.nu_ceiling),
                float(e.nu_tol), int(e.max_newton), var_ratio(td), dm_out.ptr(), _ptr(status),
                _ptr(guard))
    check(L.loghmm_reduce_mstep(_ptr(partials), _ptr(ll), B, width, _ptr(totals), *args, wptr, wlen,
                                _stream()), "loghmm_reduce_mstep")
    return totals


GUARD_STRIDE = 16  # doubles of scratch per (stream, state)


def var_ratio(td: torch.dtype) -> float:
    """Second-pass trigger for variance-type statistics: (mean shift)^2 / var
    above which the one-pass shifted sum would lose more than ~1e-11 (fp64)
    or ~1e-6 (fp32 lane partials) relative precision."""
    return 1e3 if td == torch.float64 else 10.0


def mstep(dm_in: DeviceModel, totals: torch.Tensor, n_sequences: int, config,
          dm_out: DeviceModel, status: torch.Tensor, guard: torch.Tensor,
          td: torch.dtype = torch.float64) -> None:
    L = lib()
    e = config.ecme
    check(
        L.loghmm_mstep(dm_in.ptr(), _ptr(totals), n_sequences, float(config.collapse_epsilon),
                       float(e.nu_ceiling), float(e.nu_tol), int(e.max_newton), var_ratio(td),
                       dm_out.ptr(), _ptr(status), _ptr(guard), _stream()),
        "loghmm_mstep",
    )


def variance_pass(batch: Batch, dm_out: DeviceModel, gamma: torch.Tensor, stream_index: int,
                  guard: torch.Tensor, status: torch.Tensor) -> None:
    L = lib()
    K = dm_out.K
    y = batch.y0 if stream_index == 0 else batch.y1
    need = int(L.loghmm_guard_workspace_bytes(K, batch.N))
    wptr, wlen = _WS_GUARD.get(need, y.device)
    check(
        L.loghmm_variance_pass(_code(batch.dtype), dm_out.ptr(), _ptr(y), _ptr(gamma), batch.N, K,
                               stream_index, _ptr(guard), _ptr(status), wptr, wlen, _stream()),
        "loghmm_variance_pass",
    )


def student_guard(batch: Batch, dm_out: DeviceModel, gamma: torch.Tensor, stream_index: int,
                  n_candidates: int, guard: torch.Tensor, status: torch.Tensor,
                  need_more: torch.Tensor) -> None:
    L = lib()
    K = dm_out.K
    y = batch.y0 if stream_index == 0 else batch.y1
    need = int(L.loghmm_guard_workspace_bytes(K, batch.N))
    wptr, wlen = _WS_GUARD.get(need, y.device)
    check(
        L.loghmm_student_guard(_code(batch.dtype), dm_out.ptr(), _ptr(y), _ptr(gamma), batch.N, K,
                               stream_index, n_candidates, _ptr(guard), _ptr(status),
                               _ptr(need_more), wptr, wlen, _stream()),
        "loghmm_student_guard",
    )


def variance_partial(batch: Batch, dm_out: DeviceModel, gamma: torch.Tensor, stream_index: int,
                     guard: torch.Tensor, sums: torch.Tensor) -> None:
    """Multi-rank split of variance_pass: this rank's second-pass sums -> sums[K]."""
    L = lib()
    K = dm_out.K
    y = batch.y0 if stream_index == 0 else batch.y1
    wptr, wlen = _WS_GUARD.get(int(L.loghmm_guard_workspace_bytes(K, batch.N)), y.device)
    check(L.loghmm_variance_partial(_code(batch.dtype), dm_out.ptr(), _ptr(y), _ptr(gamma), batch.N,
                                    K, stream_index, _ptr(guard), _ptr(sums), wptr, wlen, _stream()),
          "loghmm_variance_partial")


def variance_finish(dm_out: DeviceModel, stream_index: int, guard: torch.Tensor,
                    sums: torch.Tensor, status: torch.Tensor) -> None:
    check(lib().loghmm_variance_finish(dm_out.ptr(), dm_out.K, stream_index, _ptr(guard), _ptr(sums),
                                       _ptr(status), _stream()), "loghmm_variance_finish")


def student_guard_partial(batch: Batch, dm_out: DeviceModel, gamma: torch.Tensor,
                          stream_index: int, n_candidates: int, guard: torch.Tensor,
                          sums: torch.Tensor) -> None:
    """Multi-rank split of student_guard: this rank's candidate sums ->
    sums[K * GUARD_CANDIDATES]."""
    L = lib()
    K = dm_out.K
    y = batch.y0 if stream_index == 0 else batch.y1
    wptr, wlen = _WS_GUARD.get(int(L.loghmm_guard_workspace_bytes(K, batch.N)), y.device)
    check(L.loghmm_student_guard_partial(_code(batch.dtype), _ptr(y), _ptr(gamma), batch.N, K,
                                         stream_index, n_candidates, _ptr(guard), _ptr(sums), wptr,
                                         wlen, _stream()), "loghmm_student_guard_partial")


def student_guard_select(dm_out: DeviceModel, stream_index: int, n_candidates: int,
                         guard: torch.Tensor, sums: torch.Tensor, status: torch.Tensor,
                         need_more: torch.Tensor) -> None:
    check(lib().loghmm_student_guard_select(dm_out.ptr(), dm_out.K, stream_index, n_candidates,
                                            _ptr(guard), _ptr(sums), _ptr(status), _ptr(need_more),
                                            _stream()), "loghmm_student_guard_select")


# Candidate batches of the ECME guard, as training.baum_welch issues them: the
# first launch evaluates the base and the first candidate (almost always
# accepted, so the common case is one cheap data pass), each further launch
# the next GUARD_CANDIDATES-1 halvings; the reference tries at most 60
# (distributions.py:1083), so this many launches always reach a decision (a
# launch with nothing pending exits at once).  Used where the host cannot
# poll need_more (CUDA graph capture).
GUARD_FIRST = 2
GUARD_LAUNCHES = 1 + -(-(60 - (GUARD_FIRST - 1)) // (_native.GUARD_CANDIDATES - 1))


def guard_candidates(launch_index: int) -> int:
    return GUARD_FIRST if launch_index == 0 else _native.GUARD_CANDIDATES


def ext_fit(batch: Batch, dm_out: DeviceModel, gamma: torch.Tensor, stream_index: int,
            guard: torch.Tensor, status: torch.Tensor, need_more: torch.Tensor,
            poll: bool = True) -> None:
    """Weighted-sample fits of the families 6..15 left pending by the M-step
    (loghmm_ext_fit_pass, one data pass per call).  poll=True reads need_more
    after each pass (host loop); poll=False enqueues the maximum number of
    passes (a pass with nothing pending exits at once; CUDA-graph safe)."""
    L = lib()
    K = dm_out.K
    y = batch.y0 if stream_index == 0 else batch.y1
    wptr, wlen = _WS_GUARD.get(int(L.loghmm_guard_workspace_bytes(K, batch.N)), y.device)
    for _ in range(_native.EXT_MAX_PASSES):
        if poll:
            need_more.zero_()
        check(L.loghmm_ext_fit_pass(_code(batch.dtype), dm_out.ptr(), _ptr(y), _ptr(gamma), batch.N, K,
                                    stream_index, _ptr(guard), _ptr(status), _ptr(need_more), wptr,
                                    wlen, _stream()), "loghmm_ext_fit_pass")
        if poll and int(need_more.item()) == 0:
            break
