#!/usr/bin/env python3
"""Wall time of the public drop-in calls on config 2 at full size (what a user
of loghmm.training.baum_welch / inference.posteriors / viterbi sees), next to
the device-resident pipeline step."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2605_29208_b200 as H  # noqa: E402
from paper_2605_29208_b200.configs import make_config  # noqa: E402


def wall(fn, n=3):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts), r


def main():
    dtype = sys.argv[1] if len(sys.argv) > 1 else "float32"
    cfg = make_config("c2")
    seqs = [cfg.data[b] for b in range(cfg.B)]
    out = {"dtype": dtype}
    out["posteriors_batch_s"], _ = wall(lambda: H.posteriors_batch(cfg.init, seqs, dtype=dtype))
    out["viterbi_batch_s"], _ = wall(lambda: H.viterbi_batch(cfg.init, seqs, dtype=dtype))
    tc = H.TrainingConfig(max_iterations=10, rel_tol=1e-300)
    out["baum_welch_10it_s"], (m, rep) = wall(lambda: H.baum_welch(cfg.init, seqs, tc, dtype=dtype), n=2)
    out["iterations"] = rep.iterations
    print(json.dumps(out))


if __name__ == "__main__":
    main()
