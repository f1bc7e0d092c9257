"""Swap the reference `moepredict` hot-path functions for the B200 ones.

    from paper_2511_10676_b200.integration import patch_reference
    replaced = patch_reference()          # needs `moepredict` importable

See INTEGRATION.md. Only the hot path and the widened rows are replaced
(predictor, selection, evaluation, loss, layer_norm, the synthetic teacher's
generate_dataset); the reference's host code (CLI, config, pipesim) keeps
running as is.
"""

from __future__ import annotations

import importlib


def _generate_dataset_adapter(ref_synthgen):
    """Reference TeacherSpec in, reference TraceFile out, K11 in between."""
    from . import synthgen as b2s

    def generate_dataset(teacher, n):
        r = teacher.router
        spec = b2s.TeacherSpec(b2s.RouterSpec(r.hidden_dim, r.n_experts, r.n_active, r.gate_weights),
                               transform=teacher.transform, mix_matrix=teacher.mix_matrix,
                               nonlinear_hidden=teacher.nonlinear_hidden, post_norm=teacher.post_norm,
                               noise_sigma=teacher.noise_sigma, seed=teacher.seed)
        t = b2s.generate_dataset(spec, n)
        return ref_synthgen.TraceFile(t.hidden_dim, t.n_experts, t.k, t.activations, t.true_scores, t.true_topk)
    return generate_dataset


def patch_reference(package: str = "moepredict") -> list:
    from . import core, losses, metrics, predictor
    ref_synthgen = importlib.import_module(f"{package}.synthgen")
    targets = {
        "predictor": {"predict_logits": predictor.predict_logits,
                      "predict_topk_batch": predictor.predict_topk_batch},
        "core": {"top_k_batch": core.top_k_batch, "rank_order": core.rank_order,
                 "layer_norm": core.layer_norm},
        "synthgen": {"generate_dataset": _generate_dataset_adapter(ref_synthgen)},
        "metrics": {"evaluate_predictions": metrics.evaluate_predictions},
        "losses": {"loss_and_grad": losses.loss_and_grad},
    }
    replaced = []
    for mod_name, fns in targets.items():
        mod = importlib.import_module(f"{package}.{mod_name}")
        for name, fn in fns.items():
            setattr(mod, name, fn)
            replaced.append(f"{package}.{mod_name}.{name}")
    return replaced
