#!/usr/bin/env python3
"""Benchmark: F-B + Viterbi + one Baum-Welch M-step, state-steps/s (B*T*K),
BASELINE config 2 (B=4096, T=1024, K=4 Gaussian), plus % of the HBM roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--dtype float32|float64]
  python bench.py --impl reference ...   # the reference's CPU algorithm (oracle port)

One JSON line on rank 0.  A step = one pass of the pipeline over the whole
synthetic batch: loghmm_forward_backward (log_alpha, log_beta, gamma, E-step
statistics) concurrently with loghmm_viterbi (int64 path), then the
deterministic statistics reduction and the M-step kernel.  Inputs are resident
in HBM for ``value``; ``e2e`` goes through the public Pipeline API from pinned
host memory (H2D of y, D2H of the total log-likelihood and the updated model).
L2 is flushed (256 MiB write) between timed steps.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "F-B+Viterbi state-steps/s (B·T·K) at B=4096,T=1024,K=4; % of HBM roofline"
UNIT = "state-steps/s"
WORKLOAD = "c2: B=4096 T=1024 K=4 Gaussian HMM; FB(log_alpha,log_beta,gamma,xi/stats)+Viterbi(path)+1 Baum-Welch M-step"
WORKLOADS = {
    "c2": WORKLOAD,
    "c3": "c3: B=1024 T=2048 K=3 Student-t HMM; FB+Viterbi+1 Baum-Welch M-step (ECME, likelihood guard)",
    "c4": "c4: B=2048 T=2000 K=3 Gamma+von Mises joint HMM; FB+Viterbi+1 Baum-Welch M-step (Gamma NR, kappa Newton)",
    "c5": "c5: B=64 T=65536 K=64 Poisson HMM (banded A); FB+Viterbi+1 Baum-Welch M-step",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="float32", choices=["float32", "float64"])
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5"],
                    help="BASELINE config (c2 is the headline; c3-c5 are auxiliary lines)")
    ap.add_argument("--B", type=int, default=None)
    ap.add_argument("--T", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA graph")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-slices", type=int, default=2,
                    help="host-to-device copy slices overlapped with the kernels in the e2e step")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# CPU reference (the oracle port of the reference algorithm; test infra)
# ---------------------------------------------------------------------------
def oracle_spec(model):
    """Emission spec tuples of a model for the oracle (family, *params)."""
    from paper_2605_29208_b200 import HmmModel, Joint

    out = []
    for d in model.emissions:
        if isinstance(d, Joint):
            out.append(("joint", oracle_spec(HmmModel([1.0], [[1.0]], (d.first,)))[0],
                        oracle_spec(HmmModel([1.0], [[1.0]], (d.second,)))[0]))
        else:
            out.append((d.family,) + tuple(d.params().values()))
    return out


def _cpu_seq(args):
    import loghmm_oracle as O

    y, pi, A, ems = args
    lp, la = O.model_tables(pi, A)
    lb = O.emission_matrix(ems, y)
    r = O.posteriors(lp, la, lb)  # inference.py:161 (log_alpha, log_beta, gamma)
    O.viterbi(lp, la, lb)  # inference.py:191
    K = len(pi)
    xi = np.zeros((K, K))
    for t in range(len(y) - 1):  # training.py:204-210
        xi += np.exp(r["log_alpha"][t][:, None] + la + (lb[t + 1] + r["log_beta"][t + 1])[None, :] - r["ll"])
    return r["gamma"], xi, r["gamma"][0], r["gamma"][:-1].sum(axis=0), r["ll"]


def cpu_reference_run(cfg, n_seq, pool):
    """One bounded sample of the workload on the host: per-sequence reference
    E-step + Viterbi over a process pool, then the pooled M-step."""
    import loghmm_oracle as O

    m = cfg.init
    ems = oracle_spec(m)
    seqs = [cfg.data[b % cfg.B] for b in range(n_seq)]
    t0 = time.perf_counter()
    res = pool.map(_cpu_seq, [(y, m.initial, m.transitions, ems) for y in seqs])
    G = np.concatenate([r[0] for r in res])
    Y = np.concatenate(seqs)
    for j, fam in enumerate(ems):
        if fam[0] in ("gaussian", "poisson", "gamma", "von_mises", "student_t"):
            O.fit(fam, Y, G[:, j])
    return time.perf_counter() - t0


def cpu_pool():
    import multiprocessing as mp

    sys.path.insert(0, str(ROOT / "oracle"))
    cores = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    return ctx.Pool(cores), cores


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2605_29208_b200.configs import make_config

    cfg = make_config(a.config, B=64, T=a.T)
    pool, cores = cpu_pool()
    # size each step so the whole --warmup + --steps run takes ~2 minutes
    probe = cpu_reference_run(cfg, cores, pool)
    per_seq = probe / cores
    budget = 120.0 / max(1, a.steps + a.warmup)
    n_seq = int(max(1, min(256, budget / per_seq)))
    for _ in range(a.warmup):
        cpu_reference_run(cfg, n_seq, pool)
    tot = 0.0
    for _ in range(a.steps):
        tot += cpu_reference_run(cfg, n_seq, pool)
    pool.close()
    K = cfg.K
    val = a.steps * n_seq * cfg.T * K / tot
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": val,
        "unit": UNIT,
        "n_gpus": a.gpus,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": 1000.0 * tot / a.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE config 2 draw, seed 0)",
        "config": {"workload": WORKLOADS[a.config], "B": make_config(a.config).B if a.config != "c2" else 4096,
                   "T": cfg.T, "K": K, "sample_per_step": f"{n_seq} sequences x T={cfg.T}"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{n_seq} sequences of config {a.config[1]} per step (reference E-step + Viterbi per sequence over {cores} processes, pooled M-step)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks (NVML sampled during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self.nv = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def ours(a):
    import torch
    import torch.distributed as dist

    from paper_2605_29208_b200.configs import make_config
    from paper_2605_29208_b200.pipeline import Pipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist.group.WORLD
    cfg = make_config(a.config, B=a.B, T=a.T, seed=rank)  # weak scaling: each rank its own batch
    B, T, K = cfg.B, cfg.T, cfg.K
    td = torch.float32 if a.dtype == "float32" else torch.float64
    esz = 4 if td == torch.float32 else 8
    p = Pipeline(cfg.init, B, T, a.dtype, process_group=pg)
    y_host = torch.from_numpy(cfg.data).to(td).pin_memory()
    p.load(y_host)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    for _ in range(max(3, a.warmup)):
        p.run()
    torch.cuda.synchronize()

    # ---- device-resident timing ------------------------------------------
    # One pipeline step (Viterbi || forward-backward, fused reduction + M-step,
    # variance pass) is captured once as a CUDA graph and replayed, so host
    # launch overhead stays off the device timeline; the events bracket the
    # replay on the capturing stream.  --no-graph times eager launches.
    graph = None
    if not a.no_graph:
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                p.run()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                p.run()
            graph.replay()
            torch.cuda.synchronize()
        except Exception as exc:  # capture unsupported here: eager launches
            print(f"[bench] CUDA graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    if pg is not None:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        for i in range(a.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record()
            if graph is not None:
                graph.replay()
            else:
                p.run()
            ev[i][1].record()
        torch.cuda.synchronize()
    if pg is not None:
        dist.barrier()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    # per-kernel durations (eager, events on each kernel's own stream), after
    # the timed region
    kfb, kvit = [], []
    for i in range(min(a.steps, 10)):
        flush.fill_(i & 0xFF)
        p.run(time_kernels=True)
        p.ev["fb"][1].synchronize()
        p.ev["vit"][1].synchronize()
        km = p.kernel_ms()
        kfb.append(km["fb"])
        kvit.append(km["vit"])
    torch.cuda.synchronize()
    step_ms = sum(s.elapsed_time(e) for s, e in ev) / a.steps
    t_local = torch.tensor([step_ms], device="cuda", dtype=torch.float64)
    if pg is not None:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    step_ms = float(t_local.item())
    state_steps = B * T * K * world
    value = state_steps / (step_ms / 1000.0)

    # ---- end-to-end through the public API from pinned host memory ---------
    host_out = torch.empty(p.dm_next.buf.numel(), dtype=torch.uint8).pin_memory()
    host_ll = torch.empty(1, dtype=torch.float64).pin_memory()
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]

    def e2e_step():
        # H2D of the step's observations (sliced, overlapped with the kernels
        # of the slices already on the device), the pipeline, D2H of the
        # total log-likelihood and the updated model
        p.run_from_host(y_host, slices=a.e2e_slices)
        host_ll.copy_(p.totals[-1:], non_blocking=True)
        host_out.copy_(p.dm_next.buf, non_blocking=True)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    e2e_graph = None
    if graph is not None:  # same launch mode as the device-resident timing
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                e2e_step()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            e2e_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(e2e_graph):
                e2e_step()
            e2e_graph.replay()
            torch.cuda.synchronize()
        except Exception as exc:
            print(f"[bench] e2e graph capture failed ({exc}); eager e2e", file=sys.stderr)
            e2e_graph = None
            torch.cuda.synchronize()
    for i in range(a.steps):
        flush.fill_(i & 0xFF)
        e2e_ev[i][0].record()
        if e2e_graph is not None:
            e2e_graph.replay()
        else:
            e2e_step()
        e2e_ev[i][1].record()
    torch.cuda.synchronize()
    e2e_ms = sum(s.elapsed_time(e) for s, e in e2e_ev) / a.steps
    t_local = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
    if pg is not None:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    e2e_ms = float(t_local.item())
    # sanity: the fetched result is the device result
    total_ll = float(host_ll.item())
    assert math.isfinite(total_ll)

    if rank != 0:
        if pg is not None:
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    fb_ms = statistics.mean(kfb)
    vit_ms = statistics.mean(kvit)
    ns = cfg.init.n_streams
    fb_bytes = B * T * (ns * esz + 3 * K * esz)  # y read once; log_alpha, log_beta, gamma written
    m1_bytes = B * T * (ns * esz + 3 * K * esz + 8)  # + int64 Viterbi path
    achieved = fb_bytes / (fb_ms / 1000.0) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "fb_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(a.dtype) if a.config == "c2" else None
        except Exception:
            traffic = None
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": a.steps,
        "warmup": max(3, a.warmup),
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32" if td == torch.float32 else "f64",
        "data": "synthetic (BASELINE config 2 draw: Dirichlet transitions, means -3,-1,1,3, std U[0.5,1.5]; seed = rank)",
        "config": {"workload": WORKLOADS[a.config], "B": B, "T": T, "K": K, "l2": "flushed (256 MiB write) between timed steps",
                   "launch": "cuda graph replay" if graph is not None else "eager",
                   "parallelism": f"dp{world} (sequences sharded, statistics all-reduced)" if world > 1 else "single GPU"},
        "roofline": {
            "bound": "hbm",
            "kernel": (f"fb_large_kernel (K={K})" if K > 8 else
                       f"fb_chunk_kernel (chunk operators + meet-in-the-middle re-sweep, K={K})"
                       if td == torch.float32 and T % 8 == 0 else
                       f"fb_small_kernel (chunked associative scan, K={K})"),
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "peak_source": peak_src,
            "alg_bytes_per_launch": fb_bytes, "kernel_ms": fb_ms,
        },
        "pipeline_roofline": {
            "bytes_per_step_M1": m1_bytes, "achieved_gbs": m1_bytes / (step_ms / 1000.0) / 1e9,
            "frac": m1_bytes / (step_ms / 1000.0) / 1e9 / peak, "viterbi_kernel_ms": vit_ms,
        },
        "e2e": {"value": state_steps / (e2e_ms / 1000.0), "unit": UNIT,
                "h2d_bytes_per_step": int(y_host.numel() * esz), "d2h_bytes_per_step": 8 + int(host_out.numel()),
                "ms_per_step": e2e_ms, "h2d_slices": a.e2e_slices,
                "launch": "cuda graph replay" if e2e_graph is not None else "eager"},
        "gpu_launches": p.kernels_per_run * a.steps,
        "clocks": clk.summary(),
        "wall_s_timed_region": wall,
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        pool, cores = cpu_pool()
        cpu_cfg = make_config(a.config, B=min(64, B), T=T)
        probe = cpu_reference_run(cpu_cfg, cores, pool)
        n_seq = int(max(cores, min(512, cores * a.cpu_seconds / max(probe, 1e-3))))
        t = cpu_reference_run(cpu_cfg, n_seq, pool)
        pool.close()
        line["cpu_baseline"] = {
            "value": n_seq * T * K / t, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{n_seq} sequences of config {a.config[1]} (T={T}, K={K}): reference E-step + Viterbi per sequence over {cores} processes + pooled M-step, {t:.1f} s",
        }
    print(json.dumps(line), flush=True)
    if pg is not None:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
    else:
        ours(a)


if __name__ == "__main__":
    main()
