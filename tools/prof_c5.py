#!/usr/bin/env python3
"""Standalone timings of the large-K kernels on the config-5 shape (each API
call alone, CUDA events, L2 flushed): Viterbi (sparse / dense path) and the
forward-backward with statistics.

  python tools/prof_c5.py [--T 65536] [--B 64] [--dtype float32] [--reps 3]
"""
import argparse
import json
import os
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
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--T", type=int, default=65536)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    cfg = make_config("c5", B=a.B, T=a.T)
    batch = engine.make_batch(cfg.data, 1, a.dtype)
    dm = engine.DeviceModel.from_model(cfg.init)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {"dtype": a.dtype, "B": a.B, "T": a.T}
    if a.only in ("", "vit"):
        vo = engine.viterbi(batch, dm)
        torch.cuda.synchronize()
        out["vit_ms"] = timeit(lambda: engine.viterbi(batch, dm, out=vo), a.reps, flush)
        os.environ["LOGHMM_VL_SPARSE"] = "0"
        out["vit_dense_ms"] = timeit(lambda: engine.viterbi(batch, dm, out=vo), a.reps, flush)
        del os.environ["LOGHMM_VL_SPARSE"]
    if a.only in ("", "fb"):
        fbo = engine.forward_backward(batch, dm, stats=True)
        torch.cuda.synchronize()
        out["fb_ms"] = timeit(lambda: engine.forward_backward(batch, dm, stats=True, out=fbo), a.reps, flush)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
