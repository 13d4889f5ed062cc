#!/usr/bin/env python3
"""Small-case check of both forward-backward decompositions against the oracle."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import loghmm_oracle as O  # noqa: E402
import paper_2605_29208_b200 as H  # noqa: E402


def main():
    algo = sys.argv[1] if len(sys.argv) > 1 else "mitm"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    os.environ["LOGHMM_FB_ALGO"] = algo
    rng = np.random.default_rng(1)
    K = 4
    pi = rng.dirichlet(np.ones(K))
    A = rng.dirichlet(np.ones(K), size=K) * 0.5 + 0.5 * np.eye(K)
    A /= A.sum(1, keepdims=True)
    m = H.HmmModel(pi, A, tuple(H.Gaussian(float(rng.normal(0, 2)), 1.0) for _ in range(K)))
    data = rng.normal(0, 2, (B, T))
    print("launching", algo, B, T, flush=True)
    r = H.posteriors_batch(m, data, check=False)
    torch.cuda.synchronize()
    print("done", flush=True)
    lp, la = O.model_tables(pi, A)
    worst = 0.0
    for b in range(B):
        o = O.posteriors(lp, la, O.emission_matrix([("gaussian", d.mu, d.sigma) for d in m.emissions], data[b]))
        s = slice(b * T, (b + 1) * T)
        worst = max(worst, abs(r.log_likelihood[b].item() - o["ll"]),
                    float(np.abs(r.gamma[s].cpu().numpy() - o["gamma"]).max()),
                    float(np.abs(r.log_alpha[s].cpu().numpy() - o["log_alpha"]).max()),
                    float(np.abs(r.log_beta[s].cpu().numpy() - o["log_beta"]).max()))
    print("worst abs diff", worst)


if __name__ == "__main__":
    main()
