"""Data-parallel Baum-Welch across ranks.

Sequences are independent in the E-step (training.py:187 loops over them),
so the batch is sharded by contiguous sequence ranges, one rank per GPU.
The only exchange per EM iteration is one all-reduce (sum) of the fp64
statistics vector produced by loghmm_reduce_stats (xi totals, gamma totals,
first-gamma sums, per-state family sums, total LL); the M-step is then
replicated on every rank.  Error semantics need the *first* offending
sequence in global order, which is one all-reduce (min) of a global index.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["shard_range", "allreduce_totals", "first_bad_sequence"]


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of n sequences for `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def allreduce_totals(totals: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-rank statistics vector in place (fp64)."""
    if totals.dtype != torch.float64:
        raise TypeError("statistics are reduced in fp64")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(totals, op=dist.ReduceOp.SUM, group=group)
    return totals


def first_bad_sequence(flags: np.ndarray, ll: np.ndarray, offset: int, device, group=None) -> int:
    """Global index of the first sequence with a dead observation or an
    infeasible likelihood (training.py:189-197 order), or -1."""
    bad = np.nonzero((flags[:, 0] >= 0) | (ll == -np.inf))[0]
    local = int(bad[0]) + offset if bad.size else np.iinfo(np.int64).max
    t = torch.tensor([local], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    v = int(t.item())
    return -1 if v == np.iinfo(np.int64).max else v
