import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch
import paper_2605_29208_b200 as H
import loghmm_oracle as O
from test_gpu_parity import _banded_model, to_tuples
for K in (64,):
  for variant in ("band", "dead"):
    for sparse in ("1", "0"):
        os.environ["LOGHMM_FBL_SPARSE"] = sparse
        rng = np.random.default_rng(1700 + K)
        m = _banded_model(rng, K, 4, dead_first=variant == "dead")
        seqs = [rng.poisson(6.0, n).astype(float) for n in (1, 2, 17, 40, 700)]
        r = H.posteriors_batch(m, seqs, dtype="float32", include_xi=True)
        g = r.gamma.cpu().numpy(); la = r.log_alpha.cpu().numpy(); lb = r.log_beta.cpu().numpy()
        with np.errstate(divide="ignore"):
            lp, lA = O.model_tables(m.initial, m.transitions)
        for b in range(len(seqs)):
            s = slice(r.offsets[b], r.offsets[b + 1])
            with np.errstate(invalid="ignore", divide="ignore"):
                o = O.posteriors(lp, lA, O.emission_matrix(to_tuples(m), seqs[b]), include_xi=True)
            nanrows = np.where(np.isnan(g[s]).any(1))[0]
            print(K, variant, sparse, b, len(seqs[b]), "ll", r.log_likelihood[b].item(), o["ll"], "nan gamma rows", nanrows[:6], len(nanrows),
                  "ref nan", np.isnan(o["gamma"]).sum(), "maxdiff", np.nanmax(np.abs(g[s] - o["gamma"])))
