#!/usr/bin/env python3
"""Per-kernel timing of the config-2 hot path, each kernel launched alone
(CUDA events on the launching stream, L2 flushed between launches).

  python tools/prof_kernels.py [--dtype float32] [--reps 20] [--only fb|vit|small]
"""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2605_29208_b200 import engine  # noqa: E402
from paper_2605_29208_b200.configs import make_config  # noqa: E402


def timeit(fn, reps, flush):
    evs = []
    for i in range(reps):
        flush.fill_(i & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        evs.append((s, e))
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in evs)
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    ap.add_argument("--B", type=int, default=4096)
    ap.add_argument("--T", type=int, default=1024)
    a = ap.parse_args()
    cfg = make_config("c2", B=a.B, T=a.T)
    batch = engine.make_batch(cfg.data, 1, a.dtype)
    dm = engine.DeviceModel.from_model(cfg.init)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fbo = engine.forward_backward(batch, dm, stats=True)
    vo = engine.viterbi(batch, dm)
    torch.cuda.synchronize()
    out = {"dtype": a.dtype, "B": a.B, "T": a.T}
    if a.only in ("", "fb"):
        out["fb_ms"] = timeit(lambda: engine.forward_backward(batch, dm, stats=True, out=fbo), a.reps, flush)
        out["fb_nostats_noout_ms"] = timeit(
            lambda: engine.forward_backward(batch, dm, alpha=False, beta=False, gamma=False), a.reps, flush)
    if a.only in ("", "fb", "fbm") and hasattr(engine.lib(), "loghmm_fb_mstep"):
        from paper_2605_29208_b200.training import TrainingConfig
        tc = TrainingConfig()
        tot = torch.empty(fbo.partials.shape[1] + 1, dtype=torch.float64, device="cuda")
        dm2 = engine.DeviceModel.from_model(cfg.init)
        st = torch.zeros(2 * dm.K, dtype=torch.int32, device="cuda")
        gd = torch.zeros(2 * dm.K * engine.GUARD_STRIDE, dtype=torch.float64, device="cuda")
        ws = engine.Workspace()
        out["fb_mstep_ms"] = timeit(lambda: engine.fb_mstep(batch, dm, fbo, tot, tc, dm2, st, gd, ws),
                                    a.reps, flush)
    if a.only in ("", "vit"):
        out["vit_ms"] = timeit(lambda: engine.viterbi(batch, dm, out=vo), a.reps, flush)
    if a.only in ("", "small"):
        from paper_2605_29208_b200.training import TrainingConfig
        tc = TrainingConfig()
        tot = torch.empty(fbo.partials.shape[1] + 1, dtype=torch.float64, device="cuda")
        dm2 = engine.DeviceModel.from_model(cfg.init)
        st = torch.zeros(2 * dm.K, dtype=torch.int32, device="cuda")
        gd = torch.zeros(2 * dm.K * engine.GUARD_STRIDE, dtype=torch.float64, device="cuda")
        ws = engine.Workspace()
        out["reduce_stats_ms"] = timeit(lambda: engine.reduce_stats(fbo.partials, fbo.ll, tot), a.reps, flush)
        out["reduce_only_ms"] = timeit(
            lambda: engine.reduce_mstep(fbo.partials, fbo.ll, tot, workspace=ws), a.reps, flush)
        out["reduce_mstep_ms"] = timeit(
            lambda: engine.reduce_mstep(fbo.partials, fbo.ll, tot, dm, a.B, tc, dm2, st, gd,
                                        workspace=ws), a.reps, flush)
        out["mstep_ms"] = timeit(lambda: engine.mstep(dm, tot, a.B, tc, dm2, st, gd), a.reps, flush)
        out["variance_pass_ms"] = timeit(
            lambda: engine.variance_pass(batch, dm2, fbo.gamma, 0, gd, st), a.reps, flush)
    esz = 4 if a.dtype == "float32" else 8
    K = 4
    if "fb_ms" in out:
        out["fb_gbs"] = a.B * a.T * (esz + 3 * K * esz) / out["fb_ms"] / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
