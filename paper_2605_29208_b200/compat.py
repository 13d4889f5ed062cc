"""Drop-in shim for the reference package itself (``loghmm``).

The reference's operator interface for an emission is its family tag plus a
parameter record (``Distribution.family`` / ``params()``,
/root/reference/pkg/src/loghmm/distributions.py:164-184, and the ``FAMILIES``
registry :540-559).  This module accepts the reference's own ``HmmModel`` and
distribution objects by duck typing on exactly that interface, runs the hot
path on the B200 core, and hands back the reference's own result types:

    import loghmm
    from paper_2605_29208_b200 import compat
    handle = compat.install(loghmm)      # rebinds the hot path
    loghmm.posteriors(model, seq)        # -> loghmm.inference.ForwardBackwardResult (GPU)
    loghmm.baum_welch(model, data)       # -> (loghmm.HmmModel, loghmm.training.TrainingReport)
    handle.uninstall()

Rebound entry points (the functions SURVEY.md §8(b) lists for the path):
``inference.emission_log_matrix`` (:122), ``forward_log`` (:148),
``backward_log`` (:154), ``posteriors`` (:161), ``viterbi`` (:191),
``training.baum_welch`` (:160) and ``training.score_model`` (:89), plus the
package-level re-exports.  Exceptions and warnings are re-raised as the
reference's own classes (``InfeasibleSequenceError``, ``TrainingError``,
``FitWarning``) with the same messages.  A family the device does not
evaluate raises NotImplementedError -- the shim never falls back to the CPU.
"""

from __future__ import annotations

import functools
import warnings

import numpy as np

from . import distributions as D
from . import inference as I
from . import training as Tr

__all__ = ["to_device_model", "to_device_distribution", "install", "Installed"]


def to_device_distribution(dist) -> D.Distribution:
    """A drop-in distribution from any object with ``family`` and ``params()``
    (the reference's Distribution interface)."""
    if isinstance(dist, D.Distribution):
        return dist
    fam = getattr(dist, "family", None)
    ctor = D.FAMILIES.get(fam)
    if ctor is None:
        raise NotImplementedError(f"emission family '{fam}' is not on the B200 path")
    p = dist.params()
    if fam == "categorical":
        return ctor(tuple(p[f"p{k}"] for k in range(len(p))))
    return ctor(*p.values())


def to_device_model(model) -> I.HmmModel:
    """A drop-in HmmModel from the reference's (``initial``, ``transitions``,
    ``emissions``)."""
    if isinstance(model, I.HmmModel):
        return model
    return I.HmmModel(np.asarray(model.initial, dtype=float), np.asarray(model.transitions, dtype=float),
                      tuple(to_device_distribution(d) for d in model.emissions))


def _to_reference_distribution(ref_cls, dist):
    p = dist.params()
    if getattr(ref_cls, "family", None) == "categorical":
        return ref_cls(tuple(p[f"p{k}"] for k in range(len(p))))
    return ref_cls(*p.values())


class Installed:
    """Handle returned by ``install``: the rebound names and their originals."""

    def __init__(self, pkg, saved):
        self.pkg = pkg
        self.saved = saved

    def uninstall(self) -> None:
        for (mod, name), fn in self.saved.items():
            setattr(mod, name, fn)


def install(pkg, dtype: str = "float64") -> Installed:
    """Rebind the hot-path entry points of the reference package ``pkg``
    (``import loghmm``) to the B200 core."""
    inf = pkg.inference
    trn = pkg.training
    dst = pkg.distributions
    RefFB, RefVit = inf.ForwardBackwardResult, inf.ViterbiResult
    RefInfeasible = inf.InfeasibleSequenceError
    RefTrainingError, RefReport, RefScore = trn.TrainingError, trn.TrainingReport, trn.ModelScore
    RefFitWarning = dst.FitWarning

    def translate(fn):
        """Map the drop-in's exceptions / warnings onto the reference's classes."""

        @functools.wraps(fn)
        def wrapper(*a, **k):
            with warnings.catch_warnings(record=True) as caught:
                warnings.simplefilter("always")
                try:
                    out = fn(*a, **k)
                except I.InfeasibleSequenceError as exc:
                    raise RefInfeasible(str(exc)) from exc
                except Tr.TrainingError as exc:
                    raise RefTrainingError(str(exc)) from exc
            for w in caught:
                cat = RefFitWarning if issubclass(w.category, D.FitWarning) else w.category
                warnings.warn(str(w.message), cat, stacklevel=2)
            return out

        return wrapper

    @translate
    def emission_log_matrix(model, sequence):
        return np.asarray(I.emission_log_matrix(to_device_model(model), inf.validate_sequence(sequence), dtype))

    @translate
    def forward_log(model, sequence):
        return I.forward_log(to_device_model(model), inf.validate_sequence(sequence), dtype)

    @translate
    def backward_log(model, sequence):
        return I.backward_log(to_device_model(model), inf.validate_sequence(sequence), dtype)

    @translate
    def posteriors(model, sequence, include_xi=False):
        r = I.posteriors(to_device_model(model), inf.validate_sequence(sequence), include_xi, dtype)
        return RefFB(log_alpha=r.log_alpha, log_beta=r.log_beta, log_likelihood=r.log_likelihood,
                     gamma=r.gamma, xi=r.xi)

    @translate
    def viterbi(model, sequence):
        r = I.viterbi(to_device_model(model), inf.validate_sequence(sequence), dtype)
        return RefVit(path=r.path, log_joint=r.log_joint)

    @translate
    def baum_welch(model, data, config=None):
        dm = to_device_model(model)
        cfg = None
        if config is not None:
            e = config.ecme
            cfg = Tr.TrainingConfig(max_iterations=config.max_iterations, rel_tol=config.rel_tol,
                                    collapse_epsilon=config.collapse_epsilon,
                                    ecme=D.EcmeConfig(e.nu_ceiling, e.nu_tol, e.max_newton))
        if isinstance(data, np.ndarray) and data.ndim == 1:
            data = [data]
        seqs = [inf.validate_sequence(s) for s in data]
        if not seqs:
            raise RefTrainingError("training data contains no sequences")
        fitted, rep = Tr.baum_welch(dm, seqs, cfg, dtype)
        ems = []
        for orig, conv, new in zip(model.emissions, dm.emissions, fitted.emissions):
            # a collapsed state keeps its object (training.py:139-141)
            ems.append(orig if new is conv else _to_reference_distribution(type(orig), new))
        out = model if fitted is dm else type(model)(fitted.initial, fitted.transitions, tuple(ems))
        return out, RefReport(log_likelihood_trace=rep.log_likelihood_trace, iterations=rep.iterations,
                              converged=rep.converged, collapsed_states=rep.collapsed_states)

    @translate
    def score_model(model, data):
        if isinstance(data, np.ndarray) and data.ndim == 1:
            data = [data]
        s = Tr.score_model(to_device_model(model), [inf.validate_sequence(x) for x in data], dtype)
        return RefScore(s.log_likelihood, s.num_params, s.num_obs, s.aic, s.bic, s.aicc)

    new = {"emission_log_matrix": emission_log_matrix, "forward_log": forward_log,
           "backward_log": backward_log, "posteriors": posteriors, "viterbi": viterbi}
    new_t = {"baum_welch": baum_welch, "score_model": score_model}
    saved = {}
    for mod, table in ((inf, new), (trn, new_t), (pkg, {**new, **new_t})):
        for name, fn in table.items():
            if hasattr(mod, name):
                saved[(mod, name)] = getattr(mod, name)
                setattr(mod, name, fn)
    return Installed(pkg, saved)
