"""Minimal dataset container for training / evaluation calls.

Mirrors the fields of the reference's TraceFile and make_dataset
(pkg/src/moepredict/synthgen.py:95-159) — the on-disk MOEPA1 format and the
synthetic teacher are outside the hot path and not rebuilt here;
any object with these attributes is accepted by train() / evaluate().
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import top_k_batch
from .exceptions import DataError


@dataclass
class TraceFile:
    hidden_dim: int
    n_experts: int
    k: int
    activations: np.ndarray  # (n, d) float32
    true_scores: np.ndarray  # (n, E) float32
    true_topk: np.ndarray    # (n, k) int64, rows ascending

    def __len__(self) -> int:
        return self.activations.shape[0]


def make_dataset(activations, true_scores, k: int) -> TraceFile:
    """Assemble a TraceFile, deriving top-k labels from the float32 scores (synthgen.py:148-159)."""
    acts = np.ascontiguousarray(np.asarray(activations), dtype=np.float32)
    scores = np.ascontiguousarray(np.asarray(true_scores), dtype=np.float32)
    if acts.ndim != 2 or scores.ndim != 2 or acts.shape[0] != scores.shape[0]:
        raise DataError("activations and scores must be (n, d) and (n, E)")
    topk = top_k_batch(scores.astype(np.float64), k) if len(acts) else np.zeros((0, k), dtype=np.int64)
    return TraceFile(acts.shape[1], scores.shape[1], k, acts, scores, topk)
