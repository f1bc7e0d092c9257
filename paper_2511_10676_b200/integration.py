"""Swap the reference `moepredict` hot-path functions for the B200 ones.

    from paper_2511_10676_b200.integration import patch_reference
    replaced = patch_reference()          # needs `moepredict` importable
    ...
    unpatch_reference()                   # restore every binding

The reference binds hot-path names at import time in several modules
(pkg/src/moepredict/__init__.py:5-118 re-exports them; metrics.py:18-20,
trainer.py:15-18 and estimator.py:14-18 import predict_logits,
loss_and_grad, forward, backward, evaluate_predictions and train by name), so
rebinding the defining module is not enough: every module of the package
whose attribute IS the original function object is rebound.

Replacements keep the reference's contract at the boundary: numpy in, the
reference's own result classes out (EvalResult, ExpertSelection,
PredictorModel, TrainingReport, TraceFile), and errors raised as the
reference's exception classes (moepredict.exceptions) with the same messages.
The reference's host code (CLI, config, pipesim, its optimizer class) keeps
running as is. See INTEGRATION.md.
"""

from __future__ import annotations

import dataclasses
import functools
import importlib
import sys

from .exceptions import MoePredictError

_SAVED: list = []  # (module, attribute, original) of every rebinding, for unpatch_reference


def _reraise_as_reference(ref_exc):
    def deco(fn):
        @functools.wraps(fn)
        def wrapped(*args, **kw):
            try:
                return fn(*args, **kw)
            except MoePredictError as e:
                cls = getattr(ref_exc, type(e).__name__, None)
                if cls is None:
                    raise
                raise cls(str(e)) from e
        return wrapped
    return deco


def _adapters(package: str) -> dict:
    """(defining module, name) -> replacement callable."""
    from . import core, losses, metrics, predictor, synthgen as b2s, trainer
    R = {m: importlib.import_module(f"{package}.{m}")
         for m in ("core", "predictor", "losses", "metrics", "trainer", "synthgen", "exceptions")}
    wrap = _reraise_as_reference(R["exceptions"])

    def to_ref_eval(res):
        return R["metrics"].EvalResult(**{f.name: getattr(res, f.name) for f in dataclasses.fields(res)})

    def to_ref_model(m):
        kw = {f.name: getattr(m, f.name) for f in dataclasses.fields(m) if f.name not in ("_cache",)}
        return R["predictor"].PredictorModel(**kw)

    def predict_topk(model, x, m):
        sel = predictor.predict_topk(model, x, m)
        return R["core"].ExpertSelection(indices=sel.indices, raw_scores=sel.raw_scores)

    def evaluate_predictions(logits, true_topk, n_experts, m_list=None, true_scores=None):
        return to_ref_eval(metrics.evaluate_predictions(logits, true_topk, n_experts, m_list, true_scores))

    def evaluate(model, trace, m_list=None):
        return to_ref_eval(metrics.evaluate(model, trace, m_list))

    def train(config, data):
        model, rep = trainer.train(config, data)
        epochs = [R["trainer"].EpochStats(**dataclasses.asdict(e)) for e in rep.epochs]
        return to_ref_model(model), R["trainer"].TrainingReport(epochs, rep.overprov_m)

    def generate_dataset(teacher, n):
        r = teacher.router
        spec = b2s.TeacherSpec(b2s.RouterSpec(r.hidden_dim, r.n_experts, r.n_active, r.gate_weights),
                               transform=teacher.transform, mix_matrix=teacher.mix_matrix,
                               nonlinear_hidden=teacher.nonlinear_hidden, post_norm=teacher.post_norm,
                               noise_sigma=teacher.noise_sigma, seed=teacher.seed)
        t = b2s.generate_dataset(spec, n)
        return R["synthgen"].TraceFile(t.hidden_dim, t.n_experts, t.k, t.activations, t.true_scores, t.true_topk)

    return {
        ("predictor", "predict_logits"): wrap(predictor.predict_logits),          # predictor.py:330-334
        ("predictor", "predict_topk_batch"): wrap(predictor.predict_topk_batch),  # predictor.py:347-351
        ("predictor", "predict_topk"): wrap(predict_topk),                        # predictor.py:337-344
        ("predictor", "forward"): wrap(predictor.forward),                        # predictor.py:243-258
        ("predictor", "backward"): wrap(predictor.backward),                      # predictor.py:300-327
        ("core", "top_k"): wrap(core.top_k),                                      # core.py:27-39
        ("core", "top_k_batch"): wrap(core.top_k_batch),                          # core.py:42-48
        ("core", "rank_order"): wrap(core.rank_order),                            # core.py:51-54
        ("core", "layer_norm"): wrap(core.layer_norm),                            # core.py:57-68
        ("core", "softmax"): wrap(core.softmax),                                  # core.py:19-24
        ("losses", "loss_and_grad"): wrap(losses.loss_and_grad),                  # losses.py:243-273
        ("losses", "weighted_bce_loss"): wrap(losses.weighted_bce_loss),          # losses.py:143-153
        ("losses", "focal_loss"): wrap(losses.focal_loss),                        # losses.py:156-179
        ("losses", "ranking_hinge"): wrap(losses.ranking_hinge),                  # losses.py:182-217
        ("losses", "ranking_aware_loss"): wrap(losses.ranking_aware_loss),        # losses.py:220-240
        ("metrics", "evaluate_predictions"): wrap(evaluate_predictions),          # metrics.py:138-193
        ("metrics", "evaluate"): wrap(evaluate),                                  # metrics.py:196-207
        ("trainer", "train"): wrap(train),                                        # trainer.py:131-204
        ("synthgen", "generate_dataset"): wrap(generate_dataset),                 # synthgen.py:162-189
    }


def patch_reference(package: str = "moepredict") -> list:
    """Rebind every hot-path name of `package` (in every module that holds it)
    to the B200 implementation. Returns the rebound 'module.attr' names."""
    importlib.import_module(package)
    for m in ("core", "predictor", "losses", "metrics", "trainer", "synthgen", "estimator"):
        importlib.import_module(f"{package}.{m}")
    repl = _adapters(package)
    originals = {}
    for (mod_name, name), fn in repl.items():
        orig = getattr(importlib.import_module(f"{package}.{mod_name}"), name)
        originals[id(orig)] = (orig, fn)
    replaced = []
    mods = [(n, m) for n, m in list(sys.modules.items())
            if m is not None and (n == package or n.startswith(package + "."))]
    for mod_name, mod in mods:
        for attr, val in list(vars(mod).items()):
            hit = originals.get(id(val))
            if hit is not None and hit[0] is val:
                _SAVED.append((mod, attr, val))
                setattr(mod, attr, hit[1])
                replaced.append(f"{mod_name}.{attr}")
    return sorted(replaced)


def unpatch_reference() -> None:
    """Restore every binding patch_reference changed (last patch first)."""
    while _SAVED:
        mod, attr, val = _SAVED.pop()
        setattr(mod, attr, val)
