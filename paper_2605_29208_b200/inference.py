"""Drop-in for the reference inference layer (inference.py), batched on B200.

Same names, argument meanings, result types and error messages as
/root/reference/pkg/src/loghmm/inference.py; the numbers come from the
sm_100a kernels:

  emission_log_matrix  inference.py:122   -> loghmm_emission
  forward_log          inference.py:149   -> loghmm_forward_backward
  backward_log         inference.py:155   -> loghmm_forward_backward
  posteriors           inference.py:161   -> loghmm_forward_backward
  viterbi              inference.py:191   -> loghmm_viterbi
  posterior_decode     inference.py:213   (argmax of gamma, first index)

Single-sequence calls take and return numpy arrays exactly like the
reference.  ``*_batch`` variants take a [B, T] array / tensor or a list of
(ragged) sequences and return device tensors in the packed [N, K] layout.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from .distributions import Distribution

__all__ = [
    "HmmModel",
    "ForwardBackwardResult",
    "ViterbiResult",
    "BatchPosteriors",
    "BatchViterbi",
    "InfeasibleSequenceError",
    "validate_sequence",
    "emission_log_matrix",
    "forward_log",
    "backward_log",
    "posteriors",
    "viterbi",
    "posterior_decode",
    "posteriors_batch",
    "viterbi_batch",
]

STOCHASTIC_TOL = 1e-12


class InfeasibleSequenceError(ValueError):
    """The observations have zero probability under the model."""


@dataclass(frozen=True, eq=False)
class HmmModel:
    """Initial distribution, row-stochastic transitions, per-state emissions
    (inference.py:39-88, same validation and messages)."""

    initial: np.ndarray
    transitions: np.ndarray
    emissions: tuple[Distribution, ...]

    def __eq__(self, other):
        if not isinstance(other, HmmModel):
            return NotImplemented
        return (
            np.array_equal(self.initial, other.initial)
            and np.array_equal(self.transitions, other.transitions)
            and self.emissions == other.emissions
        )

    def __post_init__(self):
        pi = np.asarray(self.initial, dtype=float).copy()
        a = np.asarray(self.transitions, dtype=float).copy()
        emissions = tuple(self.emissions)
        k = pi.shape[0]
        if pi.ndim != 1 or a.shape != (k, k):
            raise ValueError(f"shape mismatch: initial has {k} states, transitions {a.shape}")
        if len(emissions) != k:
            raise ValueError(f"expected {k} emission distributions, got {len(emissions)}")
        if (pi < 0).any() or (a < 0).any():
            raise ValueError("probabilities must be non-negative")
        if abs(pi.sum() - 1.0) > STOCHASTIC_TOL:
            raise ValueError(f"initial distribution sums to {pi.sum()!r}, expected 1")
        for i, row_sum in enumerate(a.sum(axis=1)):
            if abs(row_sum - 1.0) > STOCHASTIC_TOL:
                raise ValueError(f"transitions[{i}] sums to {row_sum!r}, expected 1")
        pi.setflags(write=False)
        a.setflags(write=False)
        object.__setattr__(self, "initial", pi)
        object.__setattr__(self, "transitions", a)
        object.__setattr__(self, "emissions", emissions)

    @property
    def num_states(self) -> int:
        return self.initial.shape[0]

    @property
    def n_streams(self) -> int:
        return self.emissions[0].n_streams

    def log_initial(self) -> np.ndarray:
        with np.errstate(divide="ignore"):
            return np.log(self.initial)

    def log_transitions(self) -> np.ndarray:
        with np.errstate(divide="ignore"):
            return np.log(self.transitions)


@dataclass(frozen=True)
class ForwardBackwardResult:
    log_alpha: np.ndarray
    log_beta: np.ndarray
    log_likelihood: float
    gamma: np.ndarray
    xi: np.ndarray | None = None


@dataclass(frozen=True)
class ViterbiResult:
    path: np.ndarray
    log_joint: float


@dataclass(frozen=True)
class BatchPosteriors:
    """Packed device results of posteriors_batch: per-step tensors are [N, K]
    (sequence b occupies rows offsets[b]:offsets[b+1]); xi is [N-B, K, K]."""

    log_alpha: torch.Tensor | None
    log_beta: torch.Tensor | None
    gamma: torch.Tensor | None
    log_likelihood: torch.Tensor  # [B] float64
    offsets: np.ndarray
    xi: torch.Tensor | None = None


@dataclass(frozen=True)
class BatchViterbi:
    path: torch.Tensor  # [N] int64
    log_joint: torch.Tensor  # [B] float64
    offsets: np.ndarray
    back: torch.Tensor | None = None  # [N, K] uint8 backpointers (row 0 of each sequence is 0)


def validate_sequence(values) -> np.ndarray:
    """inference.py:113-119 (host-side check for single sequences)."""
    seq = np.asarray(values, dtype=float)
    if seq.ndim != 1 or seq.shape[0] < 1:
        raise ValueError("an observation sequence must be a non-empty 1-D array")
    if np.isnan(seq).any():
        raise ValueError("observation sequence contains NaN")
    return seq


RANGE_MSG = ("the forward and backward vectors of sequence {s} are further apart than the compute "
             "precision's exponent range at some step (posteriors not representable): use dtype='float64'")


def _raise_flags(flags: np.ndarray, ll: np.ndarray | None, infeasible_msg: str | None):
    if (flags[:, 1] & 1).any():
        raise ValueError("observation sequence contains NaN")
    if ll is not None and infeasible_msg is not None:
        bad = np.nonzero(ll == -np.inf)[0]
        if bad.size:
            raise InfeasibleSequenceError(infeasible_msg)
    # (no reference counterpart: the reference computes in fp64 log space; the
    # large-K fp32 path reports the loss of range instead of returning NaN)
    rng = np.nonzero(flags[:, 1] & 4)[0]
    if rng.size:
        raise FloatingPointError(RANGE_MSG.format(s=int(rng[0])))


def _single(model: HmmModel, sequence, dtype):
    ns = model.n_streams
    if isinstance(sequence, (list, tuple)) and ns == 1:
        sequence = np.asarray(sequence, dtype=float)
    if torch.is_tensor(sequence) or isinstance(sequence, np.ndarray):
        if sequence.ndim != ns or sequence.shape[0] < 1:
            raise ValueError("an observation sequence must be a non-empty 1-D array")
    dm = engine.DeviceModel.from_model(model)
    batch = engine.make_batch(sequence, ns, dtype)
    return dm, batch


def _np(t):
    return None if t is None else t.cpu().numpy()


def emission_log_matrix(model: HmmModel, sequence, dtype="float64"):
    """T x K matrix of per-state emission log-densities (inference.py:122-126)."""
    dm, batch = _single(model, sequence, dtype)
    # validate_sequence (inference.py:113-119): the NaN check the reference
    # runs before evaluating any density
    if bool(torch.isnan(batch.y0).any()) or (batch.y1 is not None and bool(torch.isnan(batch.y1).any())):
        raise ValueError("observation sequence contains NaN")
    out = engine.emission(batch, dm)
    return out.cpu().numpy() if not torch.is_tensor(sequence) else out


def _single_state_log_prob(dist: Distribution, y, dtype):
    scalar = np.isscalar(y) or (isinstance(y, np.ndarray) and y.ndim == 0)
    arr = np.atleast_1d(np.asarray(y, dtype=float))
    if np.isnan(arr).any():
        raise ValueError("log_prob received NaN input")
    model = HmmModel([1.0], [[1.0]], (dist,))
    dm = engine.DeviceModel.from_model(model)
    if dist.n_streams == 2:
        batch = engine.make_batch(arr.reshape(-1, 2), 2, dtype)
    else:
        batch = engine.make_batch(arr.reshape(-1), 1, dtype)
    out = engine.emission(batch, dm).cpu().numpy()[:, 0]
    return float(out[0]) if scalar else out


def _fb_single(model, sequence, include_xi, dtype):
    dm, batch = _single(model, sequence, dtype)
    o = engine.forward_backward(batch, dm, xi=include_xi)
    flags = o.flags.cpu().numpy()
    ll = o.ll.cpu().numpy()
    return o, flags, ll


def forward_log(model: HmmModel, sequence, dtype="float64"):
    """Log forward variables and the sequence log-likelihood."""
    o, flags, ll = _fb_single(model, sequence, False, dtype)
    _raise_flags(flags, None, None)
    return _np(o.log_alpha), float(ll[0])


def backward_log(model: HmmModel, sequence, dtype="float64"):
    """Log backward variables; the last row is identically zero."""
    o, flags, ll = _fb_single(model, sequence, False, dtype)
    _raise_flags(flags, None, None)
    return _np(o.log_beta)


def posteriors(model: HmmModel, sequence, include_xi: bool = False, dtype="float64"):
    """Smoothed state posteriors (and pairwise posteriors on request)."""
    o, flags, ll = _fb_single(model, sequence, include_xi, dtype)
    _raise_flags(flags, ll, "sequence impossible under model")
    return ForwardBackwardResult(
        log_alpha=_np(o.log_alpha),
        log_beta=_np(o.log_beta),
        log_likelihood=float(ll[0]),
        gamma=_np(o.gamma),
        xi=_np(o.xi) if include_xi else None,
    )


def viterbi(model: HmmModel, sequence, dtype="float64"):
    """Most probable state path; ties break toward the smallest state index."""
    dm, batch = _single(model, sequence, dtype)
    o = engine.viterbi(batch, dm)
    lj = o.log_joint.cpu().numpy()
    _raise_flags(o.flags.cpu().numpy(), None, None)  # NaN (validate_sequence) first
    if lj[0] == -np.inf:
        raise InfeasibleSequenceError("no feasible path")
    return ViterbiResult(path=o.path.cpu().numpy(), log_joint=float(lj[0]))


def posterior_decode(fb) -> np.ndarray:
    """Per-time argmax of the smoothed posteriors (smallest index on ties)."""
    g = fb.gamma
    if torch.is_tensor(g):
        return torch.argmax(g, dim=1)
    return np.argmax(g, axis=1)


def posteriors_batch(model: HmmModel, data, include_xi=False, dtype="float64", *,
                     log_alpha=True, log_beta=True, gamma=True, check=True) -> BatchPosteriors:
    """Batched posteriors over B sequences (device tensors, packed layout)."""
    dm = engine.DeviceModel.from_model(model)
    batch = engine.make_batch(data, model.n_streams, dtype)
    o = engine.forward_backward(batch, dm, alpha=log_alpha, beta=log_beta, gamma=gamma,
                                xi=include_xi)
    if check:
        _raise_flags(o.flags.cpu().numpy(), o.ll.cpu().numpy(), "sequence impossible under model")
    return BatchPosteriors(o.log_alpha, o.log_beta, o.gamma, o.ll, batch.offsets_host, o.xi)


def viterbi_batch(model: HmmModel, data, dtype="float64", *, back=False,
                  check=True) -> BatchViterbi:
    """Batched Viterbi over B sequences with on-device backtrace."""
    dm = engine.DeviceModel.from_model(model)
    batch = engine.make_batch(data, model.n_streams, dtype)
    o = engine.viterbi(batch, dm, back=back)
    if check:
        _raise_flags(o.flags.cpu().numpy(), None, None)
    if check and (o.log_joint.cpu().numpy() == -np.inf).any():
        raise InfeasibleSequenceError("no feasible path")
    return BatchViterbi(o.path, o.log_joint, batch.offsets_host, o.back)
