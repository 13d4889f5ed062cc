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
    ap.add_argument("--single-dtype", action="store_true",
                    help="skip the second precision of config 2 (per_dtype)")
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
                         "sample": f"{n_seq} sequences of config {a.config[1]} per step (reference E-step + Viterbi per sequence over {cores} processes, pooled M-step)",
                         "cpu": cpu_info()},
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
def source_hash() -> str:
    """Hash of the CUDA sources + C ABI header: ties a committed ncu traffic
    capture to the build it measured (bench.py reports it only on a match)."""
    import hashlib

    h = hashlib.sha256()
    files = sorted((ROOT / "paper_2605_29208_b200" / "csrc").glob("*.cu*")) + [ROOT / "include" / "loghmm_b200.h"]
    for f in files:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def traffic_record(dtype: str, config: str):
    """Per-launch DRAM traffic of the forward-backward kernel from the ncu
    capture in profiles/ (tools/fb_traffic.py), if it measured this build."""
    for f in sorted((ROOT / "profiles").glob("r*_fb_traffic.json"), reverse=True):
        try:
            d = json.loads(f.read_text())
        except Exception:
            continue
        if d.get("build") != source_hash() or d.get("config") != config or dtype not in d:
            continue
        r = d[dtype]
        return r["dram_read"] + r["sm_write"], {"file": f"profiles/{f.name}", **r}
    return None, {"note": "no ncu traffic capture of this build in profiles/ (tools/fb_traffic.py)"}


def cpu_info() -> dict:
    """CPU model, numpy version and its enabled SIMD dispatch."""
    info = {"cores": os.cpu_count()}
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                info["model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        import numpy
        from numpy._core._multiarray_umath import __cpu_features__ as feats

        info["numpy"] = numpy.__version__
        on = [k for k, v in feats.items() if v]
        info["numpy_simd"] = [k for k in on if k.startswith(("AVX512", "AVX2", "FMA3"))][-4:] or on[-4:]
    except Exception:
        pass
    return info


def _time_steps(run, steps, flush):
    """CUDA-event times (ms) of `steps` calls of run(), L2 flushed before each."""
    import torch

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record()
        run()
        ev[i][1].record()
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in ev]


def _capture(fn, enabled):
    """fn captured as a CUDA graph (replay callable), or fn itself."""
    import torch

    if not enabled:
        return fn, False
    try:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        return g.replay, True
    except Exception as exc:  # capture unsupported here: eager launches
        print(f"[bench] CUDA graph capture failed ({exc}); timing eager launches", file=sys.stderr)
        torch.cuda.synchronize()
        return fn, False


def _kernel_times(p, flush, n):
    """Mean FB / Viterbi kernel durations inside the step (events on each
    kernel's own stream, eager launches after the timed region)."""
    import torch

    kfb, kvit = [], []
    for i in range(n):
        flush.fill_(i & 0xFF)
        p.run(time_kernels=True)
        p.ev["fb"][1].synchronize()
        p.ev["vit"][1].synchronize()
        km = p.kernel_ms()
        kfb.append(km["fb"])
        kvit.append(km["vit"])
    torch.cuda.synchronize()
    return statistics.mean(kfb), statistics.mean(kvit)


def _fb_alone_ms(p, flush, n):
    """Mean duration of the forward-backward call launched alone (no concurrent
    Viterbi kernel on the SMs), L2 flushed before each launch."""
    import torch

    from paper_2605_29208_b200 import engine

    ts = []
    for i in range(n):
        flush.fill_(i & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        engine.forward_backward(p.batch, p.dm, stats=True, out=p.fb, workspace=p.ws_fb)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.mean(ts)


def _fb_name(K, td_is_f32, T):
    import torch  # noqa: F401

    if K > 8:
        return f"fb_split_sweep_kernel + fb_post_kernel (K={K})"
    if td_is_f32 and T % 8 == 0:
        return f"fb_chunk_kernel (chunk operators + meet-in-the-middle re-sweep, K={K})"
    return f"fb_small_kernel (chunked associative scan, K={K})"


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
    ns = cfg.init.n_streams
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    peak, peak_src = peaks()

    def device_leg(dtype):
        """The step on HBM-resident inputs, captured as a CUDA graph: returns
        the pipeline, its pinned host input and the timings."""
        td = torch.float32 if dtype == "float32" else torch.float64
        esz = 4 if td == torch.float32 else 8
        p = Pipeline(cfg.init, B, T, dtype, process_group=pg)
        y_all = torch.from_numpy(cfg.data).to(td)
        if ns == 2:  # per-stream pinned buffers (contiguous: the H2D copies stay asynchronous)
            y_host = (y_all[..., 0].contiguous().pin_memory(), y_all[..., 1].contiguous().pin_memory())
        else:
            y_host = y_all.pin_memory()
        p.load(y_host)
        torch.cuda.synchronize()
        for _ in range(max(3, a.warmup)):
            p.run()
        torch.cuda.synchronize()
        run, graphed = _capture(p.run, not a.no_graph)
        if pg is not None:
            dist.barrier()
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        with ClockSampler(local) as clk:
            ts = _time_steps(run, a.steps, flush)
        if pg is not None:
            dist.barrier()
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        fb_ms, vit_ms = _kernel_times(p, flush, min(a.steps, 10))
        fb_alone_ms = _fb_alone_ms(p, flush, min(a.steps, 10))
        step_ms = sum(ts) / len(ts)
        t_local = torch.tensor([step_ms], device="cuda", dtype=torch.float64)
        if pg is not None:
            dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        step_ms = float(t_local.item())
        fb_bytes = B * T * (ns * esz + 3 * K * esz)  # y read once; log_alpha, log_beta, gamma written
        m1_bytes = B * T * (ns * esz + 3 * K * esz + 8)  # + int64 Viterbi path
        achieved = fb_bytes / (fb_ms / 1000.0) / 1e9
        traffic, traffic_src = traffic_record(dtype, a.config)
        leg = {
            "dtype": "f32" if esz == 4 else "f64",
            "ms_per_step": step_ms,
            "value": B * T * K * world / (step_ms / 1000.0),
            "launch": "cuda graph replay" if graphed else "eager",
            "roofline": {
                "bound": "hbm", "kernel": _fb_name(K, esz == 4, T),
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                "alg_bytes_per_launch": fb_bytes, "kernel_ms": fb_ms,
                # the same launch with the SMs to itself (inside the step it shares
                # them with the concurrent Viterbi kernel)
                "kernel_alone_ms": fb_alone_ms,
                "frac_alone": fb_bytes / (fb_alone_ms / 1000.0) / 1e9 / peak,
            },
            "pipeline_roofline": {
                "bytes_per_step_M1": m1_bytes, "achieved_gbs": m1_bytes / (step_ms / 1000.0) / 1e9,
                "frac": m1_bytes / (step_ms / 1000.0) / 1e9 / peak, "viterbi_kernel_ms": vit_ms,
            },
            "clocks": clk.summary(),
            "wall_s_timed_region": wall,
        }
        return p, y_host, leg, esz

    p, y_host, leg, esz = device_leg(a.dtype)
    h2d_bytes = int(sum(t.numel() for t in y_host) * esz) if isinstance(y_host, tuple) else int(y_host.numel() * esz)
    state_steps = B * T * K * world

    # ---- end-to-end through the public API from pinned host memory ---------
    # H2D of the step's observations (sliced, overlapped with the kernels of
    # the slices already on the device), the pipeline, D2H of the total
    # log-likelihood and the updated model
    host_out = torch.empty(p.dm_next.buf.numel(), dtype=torch.uint8).pin_memory()
    host_ll = torch.empty(1, dtype=torch.float64).pin_memory()

    def e2e_step():
        p.run_from_host(y_host, slices=a.e2e_slices)
        host_ll.copy_(p.totals[-1:], non_blocking=True)
        host_out.copy_(p.dm_next.buf, non_blocking=True)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    e2e_run, e2e_graphed = _capture(e2e_step, not a.no_graph)
    e2e_ms = statistics.mean(_time_steps(e2e_run, a.steps, flush))
    total_ll = float(host_ll.item())
    assert math.isfinite(total_ll)

    # ---- e2e with every per-step output the reference API returns ------------
    # (ForwardBackwardResult log_alpha / log_beta / gamma and ViterbiResult
    # path, inference.py:161-210) copied back to pinned host memory each step
    td = p.td
    N = B * T
    full_host = {
        "log_alpha": torch.empty((N, K), dtype=td).pin_memory(),
        "log_beta": torch.empty((N, K), dtype=td).pin_memory(),
        "gamma": torch.empty((N, K), dtype=td).pin_memory(),
        "path": torch.empty(N, dtype=torch.int64).pin_memory(),
    }

    def e2e_full_step():
        e2e_step()
        full_host["log_alpha"].copy_(p.fb.log_alpha, non_blocking=True)
        full_host["log_beta"].copy_(p.fb.log_beta, non_blocking=True)
        full_host["gamma"].copy_(p.fb.gamma, non_blocking=True)
        full_host["path"].copy_(p.vit.path, non_blocking=True)

    e2e_full_step()
    torch.cuda.synchronize()
    full_run, _ = _capture(e2e_full_step, not a.no_graph)
    full_steps = max(3, min(a.steps, 10))
    e2e_full_ms = statistics.mean(_time_steps(full_run, full_steps, flush))
    full_d2h = sum(int(t.numel() * t.element_size()) for t in full_host.values()) + 8 + int(host_out.numel())
    t_e2e = torch.tensor([e2e_ms, e2e_full_ms], device="cuda", dtype=torch.float64)
    if pg is not None:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_ms, e2e_full_ms = (float(x) for x in t_e2e.tolist())
    del full_host

    kernels_per_run = p.kernels_per_run
    # ---- the other precision of BASELINE config 2 (same run, same box) -------
    per_dtype = {leg["dtype"]: {k: leg[k] for k in ("ms_per_step", "value", "roofline", "pipeline_roofline", "launch")}}
    if a.config == "c2" and not a.single_dtype:
        other = "float64" if a.dtype == "float32" else "float32"
        del p
        torch.cuda.empty_cache()
        _, _, leg2, _ = device_leg(other)
        per_dtype[leg2["dtype"]] = {k: leg2[k] for k in ("ms_per_step", "value", "roofline",
                                                         "pipeline_roofline", "launch", "clocks")}

    if rank != 0:
        if pg is not None:
            dist.destroy_process_group()
        return

    line = {
        "metric": METRIC,
        "value": leg["value"],
        "unit": UNIT,
        "n_gpus": world,
        "steps": a.steps,
        "warmup": max(3, a.warmup),
        "ms_per_step": leg["ms_per_step"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": leg["dtype"],
        "data": "synthetic (BASELINE config draw, seed = rank; see paper_2605_29208_b200/configs.py)",
        "config": {"workload": WORKLOADS[a.config], "B": B, "T": T, "K": K,
                   "l2": "flushed (256 MiB write) between timed steps",
                   "launch": leg["launch"],
                   "parallelism": f"dp{world} (sequences sharded, statistics all-reduced)" if world > 1 else "single GPU"},
        "roofline": leg["roofline"],
        "pipeline_roofline": leg["pipeline_roofline"],
        "per_dtype": per_dtype,
        "e2e": {"value": state_steps / (e2e_ms / 1000.0), "unit": UNIT,
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": 8 + int(host_out.numel()),
                "ms_per_step": e2e_ms, "h2d_slices": a.e2e_slices,
                "launch": "cuda graph replay" if e2e_graphed else "eager",
                "returns": "total log-likelihood + updated model"},
        "e2e_full": {"value": state_steps / (e2e_full_ms / 1000.0), "unit": UNIT,
                     "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": full_d2h,
                     "ms_per_step": e2e_full_ms, "steps": full_steps,
                     "returns": "log_alpha, log_beta, gamma, Viterbi path, total LL, updated model (inference.py:161-210)"},
        "gpu_launches": kernels_per_run * a.steps,
        "clocks": leg["clocks"],
        "wall_s_timed_region": leg["wall_s_timed_region"],
    }
    if world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(a, cfg)
    print(json.dumps(line), flush=True)
    if pg is not None:
        dist.destroy_process_group()


def cpu_baseline_leg(a, cfg):
    """The oracle port of the reference algorithm on the host cores: a bounded
    sample of the workload over all cores, plus a single-process rate."""
    from paper_2605_29208_b200.configs import make_config

    T, K = cfg.T, cfg.K
    pool, cores = cpu_pool()
    cpu_cfg = make_config(a.config, B=min(64, cfg.B), T=T)
    probe = cpu_reference_run(cpu_cfg, cores, pool)
    n_seq = int(max(cores, min(cfg.B, cores * a.cpu_seconds / max(probe, 1e-3))))
    t = cpu_reference_run(cpu_cfg, n_seq, pool)
    pool.close()
    import multiprocessing as mp

    one = mp.get_context("fork").Pool(1)
    n1 = max(1, int(n_seq / cores))
    t1 = cpu_reference_run(cpu_cfg, n1, one)
    one.close()
    info = cpu_info()
    return {
        "value": n_seq * T * K / t, "unit": UNIT, "cores": cores, "kind": "port",
        "sample": f"{n_seq} sequences of config {a.config[1]} (T={T}, K={K}): reference E-step + Viterbi per sequence over {cores} processes + pooled M-step, {t:.1f} s",
        "single_process": {"value": n1 * T * K / t1, "unit": UNIT, "sample": f"{n1} sequences, 1 process, {t1:.1f} s"},
        "cpu": info,
    }


def main():
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
    else:
        ours(a)


if __name__ == "__main__":
    main()
