"""Swap the reference `moepredict` hot-path functions for the B200 ones.

    from paper_2511_10676_b200.integration import patch_reference
    replaced = patch_reference()          # needs `moepredict` importable

See INTEGRATION.md. Only the functions on the hot path are replaced; the
reference's host code (CLI, config, synthgen, pipesim) keeps running as is.
"""

from __future__ import annotations

import importlib


def patch_reference(package: str = "moepredict") -> list:
    from . import core, losses, metrics, predictor
    targets = {
        "predictor": {"predict_logits": predictor.predict_logits,
                      "predict_topk_batch": predictor.predict_topk_batch},
        "core": {"top_k_batch": core.top_k_batch, "rank_order": core.rank_order},
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
