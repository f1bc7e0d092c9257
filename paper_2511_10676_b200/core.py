"""Selection primitives and shared types (reference: pkg/src/moepredict/core.py).

`top_k`, `top_k_batch` and `rank_order` keep the reference contract — stable
descending order, ties to the lower index, `top_k*` returned ascending
(core.py:27-54) — and run on the GPU through K7 (`moep_topk_logits`).
`softmax` and `layer_norm` run K11 kernels with numpy's reduction order
(`layer_norm` bit-identical to the reference; `softmax` to within CUDA's vs
numpy's exp ulp). numpy in -> numpy out; CUDA tensors in -> CUDA tensors out.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .engine import rank_order_device, topk_logits_device
from .exceptions import ConfigurationError

LAYER_NORM_EPS = 1e-5


def _to_device(a, dtype=torch.float64):
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype), True
    return torch.as_tensor(np.asarray(a, dtype=np.float64)).to("cuda", dtype), False


def softmax(logits, axis: int = -1):
    """Max-subtracted softmax (core.py:19-24), fp64, in numpy's reduction order
    (K11 `moep_softmax_np`; any axis is moved last first)."""
    from ._lib import check, lib, ptr
    z, is_t = _to_device(logits)
    zm = torch.movedim(z, axis, -1).contiguous()
    shape = zm.shape
    flat = zm.reshape(-1, shape[-1])
    out = torch.empty_like(flat)
    if flat.numel() > 0:
        check(lib().moep_softmax_np(ptr(flat), flat.shape[0], flat.shape[1], ptr(out),
                                    torch.cuda.current_stream(flat.device).cuda_stream), "moep_softmax_np")
    out = torch.movedim(out.reshape(shape), -1, axis)
    return out if is_t else out.cpu().numpy()


def top_k_batch(scores, k: int):
    """Row-wise top-k ids, ascending; ties to the lower index (core.py:42-48)."""
    z, is_t = _to_device(scores)
    if z.dim() != 2:
        raise ValueError(f"scores must be 2-D, got shape {tuple(z.shape)}")
    if not 1 <= k <= z.shape[1]:
        raise ValueError(f"k={k} out of range for {z.shape[1]} scores")
    ids = topk_logits_device(z, k).to(torch.int64)
    return ids if is_t else ids.cpu().numpy()


def top_k(scores, k: int):
    """1-D top_k (core.py:27-39)."""
    s = scores if isinstance(scores, torch.Tensor) else np.asarray(scores, dtype=np.float64)
    if s.ndim != 1:
        raise ValueError(f"scores must be 1-D, got shape {tuple(s.shape)}")
    if not 1 <= k <= s.shape[0]:
        raise ValueError(f"k={k} out of range for {s.shape[0]} scores")
    return top_k_batch(s[None, :], k)[0]


def rank_order(scores):
    """Full stable descending order per row (core.py:51-54)."""
    z, is_t = _to_device(scores)
    if z.dim() == 1:
        z = z[None, :]
    order = rank_order_device(z).to(torch.int64)
    return order if is_t else order.cpu().numpy()


def layer_norm(x, eps: float = LAYER_NORM_EPS):
    """Non-affine layer norm, population variance (core.py:57-68).

    K11b `moep_layer_norm_np`: numpy's reduction order (0 + pairwise_sum) and
    single roundings, so the result is bit-identical to the reference's."""
    from ._lib import check, lib, ptr
    t, is_t = _to_device(x)
    if t.shape[-1] < 2:
        raise ValueError("layer_norm needs at least 2 elements")
    shape = t.shape
    flat = t.reshape(-1, shape[-1]).contiguous()
    out = torch.empty_like(flat)
    if flat.shape[0] > 0:
        check(lib().moep_layer_norm_np(ptr(flat), flat.shape[0], flat.shape[1], float(eps), ptr(out),
                                       torch.cuda.current_stream(flat.device).cuda_stream),
              "moep_layer_norm_np")
    out = out.reshape(shape)
    return out if is_t else out.cpu().numpy()


@dataclass(frozen=True)
class ExpertSelection:
    """Predicted expert set plus its raw logits (core.py:194-211)."""

    indices: np.ndarray
    raw_scores: np.ndarray

    def __post_init__(self):
        idx = np.asarray(self.indices, dtype=np.int64)
        raw = np.asarray(self.raw_scores, dtype=np.float64)
        if idx.ndim != 1 or raw.ndim != 1:
            raise ValueError("indices and raw_scores must be 1-D")
        if len(set(idx.tolist())) != idx.shape[0]:
            raise ValueError("indices must be distinct")
        if np.any(idx < 0) or np.any(idx >= raw.shape[0]):
            raise ValueError("indices out of range")
        object.__setattr__(self, "indices", np.sort(idx))
        object.__setattr__(self, "raw_scores", raw)


__all__ = ["softmax", "top_k", "top_k_batch", "rank_order", "layer_norm", "ExpertSelection",
           "ConfigurationError"]
