"""Synthetic teacher on the GPU (reference: pkg/src/moepredict/synthgen.py:37-194).

Same API and results as the reference's `generate_dataset`: sample i draws its
activation (and noise) row from Generator(Philox(key=(seed << 64) + i))
(synthgen.py:44-47, :170-174), the teacher transform and layer norm are
applied (:176-186), and the gate softmax is cast to float32 and labelled with
its top-k (:187-188, make_dataset :148-159). The per-sample Python loop of the
reference becomes one thread per sample (K11a `moep_teacher_normals`, numpy's
Philox4x64-10 + ziggurat on the device), the layer norm K11b
`moep_layer_norm_np` (numpy's pairwise order, bit-identical), the softmax +
float32 cast + top-k K11c `moep_teacher_finish`. The teacher's GEMMs
(mix / nonlinear maps / gate) are plain fp64 GEMMs on cuBLAS.

The teacher's weight matrices (random_mix_matrix, the nonlinear maps) are
drawn once per teacher from a single sequential stream, exactly as the
reference does (numpy Generator on the host, synthgen.py:79-90); they are
parameters of the dataset, not per-sample work.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._lib import check, lib, ptr
from .data import TraceFile
from .exceptions import ConfigurationError
from .trace_io import DeviceTrace

TRANSFORMS = ("identity", "linear", "nonlinear")
_TEACHER_KEY_OFFSET = 1 << 62   # synthgen.py:41
LAYER_NORM_EPS = 1e-5


def _rng(seed: int, index: int) -> np.random.Generator:
    """Counter-based per-index stream (synthgen.py:44-47)."""
    key = ((int(seed) & 0xFFFFFFFFFFFFFFFF) << 64) + int(index)
    return np.random.Generator(np.random.Philox(key=key))


@dataclass(frozen=True)
class RouterSpec:
    """One MoE layer's gate (core.py:92-114)."""

    hidden_dim: int
    n_experts: int
    n_active: int
    gate_weights: np.ndarray  # (n_experts, hidden_dim)

    def __post_init__(self):
        if self.hidden_dim < 1 or self.n_experts < 1:
            raise ConfigurationError("hidden_dim and n_experts must be positive")
        if not 1 <= self.n_active <= self.n_experts:
            raise ConfigurationError(f"n_active={self.n_active} must be in [1, {self.n_experts}]")
        w = np.asarray(self.gate_weights, dtype=np.float64)
        if w.shape != (self.n_experts, self.hidden_dim):
            raise ConfigurationError(
                f"gate_weights shape {w.shape} != ({self.n_experts}, {self.hidden_dim})")
        if not np.all(np.isfinite(w)):
            raise ConfigurationError("gate_weights must be finite")
        object.__setattr__(self, "gate_weights", w)


@dataclass(frozen=True)
class TeacherSpec:
    """Data-generating layer standing in for real attention (synthgen.py:50-76)."""

    router: RouterSpec
    transform: str = "identity"
    mix_matrix: np.ndarray | None = None
    nonlinear_hidden: int = 64
    post_norm: bool = True
    noise_sigma: float = 0.0
    seed: int = 0

    def __post_init__(self):
        if self.transform not in TRANSFORMS:
            raise ConfigurationError(f"unknown transform {self.transform!r}")
        if self.noise_sigma < 0:
            raise ConfigurationError("noise_sigma must be >= 0")
        if self.transform == "linear":
            d = self.router.hidden_dim
            m = self.mix_matrix
            if m is None:
                m = random_mix_matrix(d, self.seed)
            m = np.asarray(m, dtype=np.float64)
            if m.shape != (d, d) or not np.all(np.isfinite(m)):
                raise ConfigurationError(f"mix_matrix must be finite ({d}, {d})")
            object.__setattr__(self, "mix_matrix", m)
        if self.transform == "nonlinear" and self.nonlinear_hidden < 1:
            raise ConfigurationError("nonlinear_hidden must be positive")


def random_mix_matrix(d: int, seed: int) -> np.ndarray:
    """synthgen.py:79-82 (one stream, drawn on the host)."""
    return _rng(seed, _TEACHER_KEY_OFFSET).standard_normal((d, d)) / np.sqrt(d)


def _nonlinear_maps(spec: TeacherSpec):
    """synthgen.py:85-90."""
    d, h = spec.router.hidden_dim, spec.nonlinear_hidden
    rng = _rng(spec.seed, _TEACHER_KEY_OFFSET + 1)
    w_in = rng.standard_normal((h, d)) / np.sqrt(d)
    w_out = rng.standard_normal((d, h)) / np.sqrt(h)
    return w_in, w_out


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


class _Teacher:
    """Device copies of one teacher's matrices."""

    def __init__(self, spec: TeacherSpec, device):
        self.spec = spec
        self.dev = torch.device(device)
        # row-major [N, K] operands of moep_dgemm_nt (C = A . B^T)
        f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(self.dev)
        self.gate = f64(spec.router.gate_weights)            # [E, d]
        self.mix = self.w_in = self.w_out = None
        if spec.transform == "linear":
            self.mix = f64(spec.mix_matrix)                   # [d, d]: x @ M^T
        elif spec.transform == "nonlinear":
            w_in, w_out = _nonlinear_maps(spec)
            self.w_in, self.w_out = f64(w_in), f64(w_out)     # [h, d], [d, h]

    def _gemm(self, a: torch.Tensor, b: torch.Tensor, tanh: bool = False) -> torch.Tensor:
        """a [M, K] . b[N, K]^T on the fp64 tensor cores (moep_dgemm_nt)."""
        c = torch.empty((a.shape[0], b.shape[0]), dtype=torch.float64, device=self.dev)
        check(lib().moep_dgemm_nt(ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(c), c.stride(0), a.shape[0],
                                  b.shape[0], a.shape[1], int(tanh), _stream(self.dev)), "moep_dgemm_nt")
        return c

    def chunk(self, first: int, n: int, acts32: torch.Tensor, scores: torch.Tensor, topk: torch.Tensor):
        """Samples first .. first+n-1 into the given output row views."""
        sp, dev = self.spec, self.dev
        d, E, k = sp.router.hidden_dim, sp.router.n_experts, sp.router.n_active
        noisy = sp.noise_sigma > 0
        x64 = torch.empty((n, d), dtype=torch.float64, device=dev)
        nz = torch.empty((n, d), dtype=torch.float64, device=dev) if noisy else None
        check(lib().moep_teacher_normals(int(sp.seed) & 0xFFFFFFFFFFFFFFFF, first, n, d, int(noisy), ptr(x64),
                                         ptr(acts32), ptr(nz), _stream(dev)), "moep_teacher_normals")
        if sp.transform == "identity":
            post = x64                                  # x.copy(): x64 is not needed afterwards
        elif sp.transform == "linear":
            post = self._gemm(x64, self.mix)
        else:
            post = self._gemm(self._gemm(x64, self.w_in, tanh=True), self.w_out)
        if noisy:
            post.add_(nz.mul_(sp.noise_sigma))          # post += sigma * noise: two roundings, as numpy
        if sp.post_norm:
            check(lib().moep_layer_norm_np(ptr(post), n, d, LAYER_NORM_EPS, ptr(post), _stream(dev)),
                  "moep_layer_norm_np")
        logits = self._gemm(post, self.gate)
        check(lib().moep_teacher_finish(ptr(logits), n, E, k, ptr(scores), ptr(topk), _stream(dev)),
              "moep_teacher_finish")


def generate_dataset_device(teacher: TeacherSpec, n: int, device="cuda", chunk_rows: int = 262144,
                            first_index: int = 0) -> DeviceTrace:
    """generate_dataset (synthgen.py:162-189) into HBM: activations fp32 [n, d],
    scores fp32 [n, E], top-k int32 [n, k] ascending."""
    if n < 1:
        raise ValueError("n must be >= 1")
    r = teacher.router
    dev = torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError("generate_dataset_device needs a CUDA device (there is no CPU fallback)")
    acts = torch.empty((n, r.hidden_dim), dtype=torch.float32, device=dev)
    scores = torch.empty((n, r.n_experts), dtype=torch.float32, device=dev)
    topk = torch.empty((n, r.n_active), dtype=torch.int32, device=dev)
    t = _Teacher(teacher, dev)
    for c0 in range(0, n, chunk_rows):
        c1 = min(n, c0 + chunk_rows)
        t.chunk(first_index + c0, c1 - c0, acts[c0:c1], scores[c0:c1], topk[c0:c1])
    return DeviceTrace(r.hidden_dim, r.n_experts, r.n_active, acts, scores, topk)


def generate_dataset(teacher: TeacherSpec, n: int, device="cuda") -> TraceFile:
    """Drop-in for the reference's generate_dataset: host TraceFile
    (activations / scores float32, top-k int64)."""
    return generate_dataset_device(teacher, n, device=device).to_host()


def expert_activation_counts(trace) -> np.ndarray:
    """synthgen.py:192-194."""
    topk = trace.true_topk
    if isinstance(topk, torch.Tensor):
        return torch.bincount(topk.reshape(-1).long(), minlength=trace.n_experts).cpu().numpy()
    return np.bincount(np.asarray(topk).ravel(), minlength=trace.n_experts)


__all__ = ["RouterSpec", "TeacherSpec", "random_mix_matrix", "generate_dataset", "generate_dataset_device",
           "expert_activation_counts", "TRANSFORMS"]
