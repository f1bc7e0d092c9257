"""Training objectives (reference: pkg/src/moepredict/losses.py).

Four families, each returning (scalar loss, d loss / d logits):
mse, wbce (two tiers), focal, ranking (three-tier WBCE + pairwise hinge).
Labels come from K3 (`moep_labels`) and the loss + gradient from K4
(`moep_loss` + `moep_loss_finalize`) on the GPU. numpy inputs run the kernels
in float64 (the reference's arithmetic, so results agree to ~1e-12); CUDA
fp32 tensors run the fp32-logit training mode (math still fp64 per element).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, dtype_code, lib, ptr
from .exceptions import ConfigurationError

FAMILIES = ("mse", "wbce", "focal", "ranking")
FAMILY_CODE = {"mse": 0, "wbce": 1, "focal": 2, "ranking": 3}
TOP_TIER_SIZE = 10
MID_TIER_SIZE = 30


@dataclass(frozen=True)
class LossSpec:
    """Loss family plus every tunable the families share (losses.py:31-53)."""

    family: str = "wbce"
    top_weight: float = 3.0
    mid_weight: float = 1.5
    rest_weight: float = 0.5
    ranking_lambda: float = 0.3
    margin: float = 0.1
    focal_gamma: float = 2.0
    focal_alpha: float = 0.25
    normalize_ranking: bool = True

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ConfigurationError(f"unknown loss family {self.family!r}")
        if min(self.top_weight, self.mid_weight, self.rest_weight) <= 0:
            raise ConfigurationError("tier weights must be positive")
        if self.ranking_lambda < 0:
            raise ConfigurationError("ranking_lambda must be >= 0")
        if self.margin <= 0:
            raise ConfigurationError("margin must be positive")


def _stream(dev):
    return torch.cuda.current_stream(dev).cuda_stream


@dataclass(frozen=True)
class BatchLabels:
    """Per-batch ground truth (losses.py:56-83): true scores, top-k mask and
    1-based stable rank. Arrays are numpy (reference layout) or CUDA tensors."""

    true_scores: object
    topk_mask: object
    rank_of: object

    @classmethod
    def from_scores(cls, true_scores, k: int) -> "BatchLabels":
        is_t = isinstance(true_scores, torch.Tensor)
        s = true_scores if is_t else torch.as_tensor(np.atleast_2d(np.asarray(true_scores, dtype=np.float64)))
        s = s.to("cuda")
        if s.dim() == 1:
            s = s[None]
        if s.dtype not in (torch.float32, torch.float64):
            s = s.to(torch.float64)
        s = s.contiguous()
        n, e = s.shape
        rank = torch.empty((n, e), dtype=torch.int32, device=s.device)
        mask = torch.empty((n, e), dtype=torch.uint8, device=s.device)
        pairs = torch.empty(n, dtype=torch.int32, device=s.device)
        check(lib().moep_labels(ptr(s), dtype_code(s), n, e, k, ptr(rank), ptr(mask), ptr(pairs), _stream(s.device)),
              "moep_labels")
        if is_t:
            return cls(s, mask.bool(), rank)
        return cls(s.cpu().numpy(), mask.bool().cpu().numpy(), rank.to(torch.int64).cpu().numpy())

    @classmethod
    def from_trace(cls, trace, rows=None) -> "BatchLabels":
        scores = trace.true_scores if rows is None else trace.true_scores[rows]
        return cls.from_scores(np.asarray(scores, dtype=np.float64), trace.k)

    @property
    def n_experts(self) -> int:
        return self.true_scores.shape[1]

    def to_device(self, dtype=torch.float64, device="cuda"):
        conv = lambda a, dt: (a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))).to(device, dt)
        return (conv(self.true_scores, dtype).contiguous(), conv(self.topk_mask, torch.uint8).contiguous(),
                conv(self.rank_of, torch.int32).contiguous())


def device_loss(spec: LossSpec, z: torch.Tensor, scores: torch.Tensor, mask_u8: torch.Tensor,
                rank_i32: torch.Tensor, n_global=None, allreduce=None, family_code=None):
    """K4 + finalize on device buffers. Returns (loss_tensor[2] fp64 on device: loss, n_pairs; dz).
    `allreduce(partial_sums_tensor)` lets data-parallel callers sum the 3 partial
    sums across ranks before the global normalisers are applied."""
    dev = z.device
    n, e = z.shape
    nblk = max(1, min(lib().moep_num_sms() * 8, (n + 7) // 8))  # enough warps to hide the per-token chains
    dz = torch.empty_like(z)
    code = FAMILY_CODE[spec.family] if family_code is None else family_code
    dzh = torch.empty_like(z) if code >= 3 else None
    partials = torch.empty((nblk, 3), dtype=torch.float64, device=dev)
    a = _lib.LossArgs()
    a.family = code
    a.top_weight, a.mid_weight, a.rest_weight = spec.top_weight, spec.mid_weight, spec.rest_weight
    a.ranking_lambda, a.margin = spec.ranking_lambda, spec.margin
    a.focal_gamma, a.focal_alpha = spec.focal_gamma, spec.focal_alpha
    a.normalize_ranking = int(spec.normalize_ranking)
    a.n, a.n_global, a.n_experts, a.dtype = n, int(n if n_global is None else n_global), e, dtype_code(z)
    a.logits, a.scores, a.rank_of, a.topk_mask = ptr(z), ptr(scores), ptr(rank_i32), ptr(mask_u8)
    a.dz, a.dz_hinge, a.partials, a.n_blocks = ptr(dz), ptr(dzh), ptr(partials), nblk
    check(lib().moep_loss(a, _stream(dev)), "moep_loss")
    if allreduce is not None:
        summed = partials.sum(dim=0, keepdim=True)
        allreduce(summed)
        partials, nblk = summed.contiguous(), 1
    out = torch.empty(2, dtype=torch.float64, device=dev)
    check(lib().moep_loss_finalize(ptr(partials), nblk, n, e, a.family, spec.ranking_lambda,
                                   int(spec.normalize_ranking), dtype_code(z), ptr(dz), ptr(dzh), ptr(out),
                                   _stream(dev)), "moep_loss_finalize")
    return out, dz


def _check_shape(pred, labels: BatchLabels):
    p = pred if isinstance(pred, torch.Tensor) else torch.as_tensor(np.atleast_2d(np.asarray(pred, dtype=np.float64)))
    if p.dim() == 1:
        p = p[None]
    if tuple(p.shape) != tuple(np.shape(labels.true_scores)):
        raise ConfigurationError(f"prediction shape {tuple(p.shape)} != labels {tuple(np.shape(labels.true_scores))}")
    return p


def loss_and_grad(spec: LossSpec, logits, labels: BatchLabels):
    """Uniform dispatch: any family -> (loss, d loss / d logits) (losses.py:243-273)."""
    is_t = isinstance(logits, torch.Tensor)
    z = _check_shape(logits, labels)
    dt = z.dtype if (is_t and z.dtype in (torch.float32, torch.float64)) else torch.float64
    z = z.to("cuda", dt).contiguous()
    scores, mask, rank = BatchLabels.to_device(labels, dt)  # any object with the three fields (the reference's too)
    out, dz = device_loss(spec, z, scores, mask, rank)
    loss = float(out[0].item())
    return (loss, dz) if is_t else (loss, dz.cpu().numpy())


def weighted_bce_loss(logits, labels: BatchLabels, *, top_weight=3.0, rest_weight=0.5):
    """Two-tier weighted BCE (losses.py:143-153)."""
    return loss_and_grad(LossSpec("wbce", top_weight=top_weight, rest_weight=rest_weight), logits, labels)


def focal_loss(logits, labels: BatchLabels, *, gamma=2.0, alpha=0.25):
    """Alpha-balanced focal loss (losses.py:156-179)."""
    return loss_and_grad(LossSpec("focal", focal_gamma=gamma, focal_alpha=alpha), logits, labels)


def ranking_aware_loss(logits, labels: BatchLabels, *, top_weight=3.0, mid_weight=1.5, rest_weight=0.5,
                       ranking_lambda=0.3, margin=0.1, normalize_ranking=True):
    """Three-tier WBCE + pairwise hinge (losses.py:220-240)."""
    spec = LossSpec("ranking", top_weight=top_weight, mid_weight=mid_weight, rest_weight=rest_weight,
                    ranking_lambda=ranking_lambda, margin=margin, normalize_ranking=normalize_ranking)
    return loss_and_grad(spec, logits, labels)


def ranking_hinge(logits, labels: BatchLabels, *, margin=0.1, normalize=True):
    """Pairwise hinge alone (losses.py:182-217): returns (total, grad, n_pairs).
    K4 family code 4 = hinge term only (lambda 1, no WBCE part)."""
    is_t = isinstance(logits, torch.Tensor)
    z = _check_shape(logits, labels).to("cuda", torch.float64).contiguous()
    scores, mask, rank = BatchLabels.to_device(labels, torch.float64)
    spec = LossSpec("ranking", ranking_lambda=1.0, margin=margin, normalize_ranking=normalize)
    out, dz = device_loss(spec, z, scores, mask, rank, family_code=4)
    o = out.cpu().numpy()
    return float(o[0]), (dz if is_t else dz.cpu().numpy()), int(o[1])


def mse_loss(pred_scores, labels: BatchLabels):
    """Squared error against the true scores, w.r.t. probabilities (losses.py:99-110).
    Small helper on device tensors (not on the training hot path)."""
    is_t = isinstance(pred_scores, torch.Tensor)
    p = _check_shape(pred_scores, labels).to("cuda", torch.float64)
    s, _, _ = BatchLabels.to_device(labels, torch.float64)
    n = p.shape[0]
    diff = s - p
    loss = float((diff * diff).sum().item() / n)
    grad = -2.0 * diff / n
    return (loss, grad) if is_t else (loss, grad.cpu().numpy())
