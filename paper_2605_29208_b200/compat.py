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
``training.baum_welch`` (:160), ``training.score_model`` (:89),
``training.default_initial_model`` (:239) and ``model_io.read_sequences``
(:150), wherever the package bound them (package re-exports, cli.py).  Exceptions and warnings are re-raised as the
reference's own classes (``InfeasibleSequenceError``, ``TrainingError``,
``FitWarning``) with the same messages.  A family the device does not
evaluate raises NotImplementedError -- the shim never falls back to the CPU.
"""

from __future__ import annotations

import functools
import sys
import warnings

import numpy as np

from . import distributions as D
from . import inference as I
from . import seqio
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

    @translate
    def default_initial_model(num_states, families, data):
        fams = [families] if isinstance(families, str) else list(families)
        dev = Tr.default_initial_model(num_states, families, data)
        ems = []
        for j, d in enumerate(dev.emissions):
            ref_cls = dst.FAMILIES[fams[j] if len(fams) > 1 else fams[0]]
            ems.append(_to_reference_distribution(ref_cls, d))
        return inf.HmmModel(dev.initial, dev.transitions, tuple(ems))

    def read_sequences(source, column=0, delimiter=","):
        return seqio.read_sequences(source, column=column, delimiter=delimiter)

    table = {"emission_log_matrix": emission_log_matrix, "forward_log": forward_log,
             "backward_log": backward_log, "posteriors": posteriors, "viterbi": viterbi,
             "baum_welch": baum_welch, "score_model": score_model,
             "default_initial_model": default_initial_model, "read_sequences": read_sequences}
    # every module of the package that bound one of these names (the CLI
    # imports them by name, cli.py:19-28) gets the drop-in
    originals = {}
    for mod in (inf, trn, pkg.model_io):
        for name in table:
            if hasattr(mod, name):
                originals.setdefault(name, getattr(mod, name))
    saved = {}
    mods = [m for n, m in list(sys.modules.items()) if m is not None and (n == pkg.__name__ or n.startswith(pkg.__name__ + "."))]
    for mod in mods:
        for name, fn in table.items():
            cur = getattr(mod, name, None)
            if cur is not None and cur is originals.get(name):
                saved[(mod, name)] = cur
                setattr(mod, name, fn)
    return Installed(pkg, saved)
