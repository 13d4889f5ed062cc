import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_29208_b200 as H
from paper_2605_29208_b200 import distributions as D
rng = np.random.default_rng(0)
y = rng.lognormal(0.5, 0.7, 500)
for fam, d0 in [("lognormal", D.LogNormal(0.0, 1.0)), ("exponential", D.Exponential(1.0)), ("rayleigh", D.Rayleigh(1.0)), ("chi_squared", D.ChiSquared(2.0)), ("weibull", D.Weibull(1.0,1.0)), ("pareto", D.Pareto(0.1, 1.0)), ("uniform", D.Uniform(0.0, 100.0))]:
    m = H.HmmModel([1.0], [[1.0]], (d0,))
    f, rep = H.baum_welch(m, [y], H.TrainingConfig(max_iterations=2, rel_tol=1e-300))
    print(fam, f.emissions[0], rep.log_likelihood_trace)
ly = np.log(y); print("lognormal expected", ly.mean(), ly.std())
print("exp expected", 1/y.mean(), "rayleigh", np.sqrt((y*y).mean()/2), "uniform", y.min(), y.max())
