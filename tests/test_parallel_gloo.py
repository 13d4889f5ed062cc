"""Multi-rank host logic on CPU (gloo, world size 2): sharding, the fp64
statistics all-reduce and the global first-error index.  The E-step
statistics are produced by the oracle per shard; the reduced totals must
equal the single-process totals (the exchange step of SURVEY.md §8e)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import loghmm_oracle as O
from paper_2605_29208_b200.parallel import allreduce_totals, first_bad_sequence, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stats(seqs, pi, A, ems):
    K = len(pi)
    xi = np.zeros((K, K))
    gt = np.zeros(K)
    g0 = np.zeros(K)
    ll = 0.0
    for y in seqs:
        r = O.estep_sequence((0, y, pi, A, ems))
        xi += r["xi"]
        gt += r["gtot"]
        g0 += r["g0"]
        ll += r["ll"]
    return np.concatenate([xi.ravel(), gt, g0, [ll]])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    K, B, T = 3, 7, 40
    pi = rng.dirichlet(np.ones(K))
    A = rng.dirichlet(np.ones(K), size=K)
    ems = [("gaussian", float(m), 1.0) for m in (-2.0, 0.0, 2.0)]
    seqs = [rng.normal(0, 2, T) for _ in range(B)]
    lo, hi = shard_range(B, rank, world)
    tot = torch.tensor(_stats(seqs[lo:hi], pi, A, ems), dtype=torch.float64)
    allreduce_totals(tot)
    flags = np.full((hi - lo, 2), -1, dtype=np.int64)
    flags[:, 1] = 0
    ll = np.zeros(hi - lo)
    if rank == 1:
        ll[-1] = -np.inf  # a bad sequence on rank 1 (global index B-1)
    if rank == 1 and hi - lo > 1:
        flags[0, 0] = 5  # dead observation at global index lo
    bad = first_bad_sequence(flags, ll, lo, "cpu")
    q.put((rank, tot.numpy(), bad, lo))
    dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (1, 7, 4096):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_allreduce_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(0)
    K, B, T = 3, 7, 40
    pi = rng.dirichlet(np.ones(K))
    A = rng.dirichlet(np.ones(K), size=K)
    ems = [("gaussian", float(m), 1.0) for m in (-2.0, 0.0, 2.0)]
    seqs = [rng.normal(0, 2, T) for _ in range(B)]
    ref = _stats(seqs, pi, A, ems)
    for rank, tot, bad, lo in res:
        np.testing.assert_allclose(tot, ref, rtol=1e-12)
        lo1, _ = shard_range(B, 1, 2)
        assert bad == lo1  # rank 1's dead observation comes first globally
