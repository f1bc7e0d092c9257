"""Synthetic predictor workloads for bench.py, the parity tests and tools/.

Two kinds of per-layer predictor, both bf16-representable so the tensor-core
path (K1) runs:

* ``random``: the reference's Kaiming init (predictor.py:139-173, init_model)
  rounded to bf16. Its accuracy is chance level (exact-match ~ 1/C(E, k)), so
  true experts rarely sit at a selection boundary.
* ``gate``: the reference's oracle-gate construction (tests/test_metrics.py:
  185-192: w1 = eps*I, w2 = 2*W_g/eps, so that silu(eps*x)/eps*2 ~ x and the
  predictor reproduces the router gate W_g), made dense so GEMM1 still does
  d*h useful multiply-adds with a realistic accumulation error: w1 = 2^-s * H
  with H the Sylvester-Hadamard matrix (entries +-1, H H^T = d I) and
  w2 = bf16(2^(s+1) / d * W_g H^T). w1 is exactly bf16; z = W_g x + O(|a|).
  The predictor then agrees with the router for ~all tokens, so the true
  experts DO sit at the k boundary, which is what a trained predictor looks
  like (93-98 % exact match) and what makes the near-tie
  fix-up cost realistic.

Activations are the hook point's x_hat (hooks.py:19,113-114): standard
normal rows through layer_norm (core.py:57-68), rounded to bf16. Ground truth
is the router's top-k of layer_norm(x) @ W_g^T (the teacher of synthgen.py,
post-norm, no transform). Everything is generated on the device from seeds.
"""

from __future__ import annotations

import numpy as np


def round_bf16(a):
    """Round float64 to the nearest bf16 value (ties to even), as float64."""
    a = np.asarray(a, dtype=np.float64)
    m, e = np.frexp(a)
    return np.ldexp(np.rint(m * 256.0), e - 8)


def hadamard(n: int) -> np.ndarray:
    """Sylvester-Hadamard matrix H[i, j] = (-1)^popcount(i & j), n a power of 2."""
    if n & (n - 1):
        raise ValueError("hadamard needs a power of two")
    i = np.arange(n)
    bits = np.bitwise_and(i[:, None], i[None, :])
    pc = np.zeros_like(bits)
    while bits.any():
        pc += bits & 1
        bits >>= 1
    return np.where(pc & 1, -1.0, 1.0)


GATE_SHIFT = 14  # w1 = 2^-14 H: |a| ~ 2.8e-3 keeps silu within 0.1 % of a/2


def gate_weights(E: int, d: int, seed: int) -> np.ndarray:
    """Router gate W_g ~ N(0, 1/d) (config.py:97-99)."""
    return np.random.default_rng(seed).standard_normal((E, d)) / np.sqrt(d)


def make_predictor(kind: str, d: int, h: int, E: int, seed: int, gate=None):
    """A bf16-exact arch2 PredictorModel of the given kind."""
    import paper_2511_10676_b200 as pb
    if kind == "random":
        m = pb.init_model("arch2", d, h, E, seed=seed)
        m.w1, m.w2 = round_bf16(m.w1), round_bf16(m.w2)
        return m
    if kind != "gate":
        raise ValueError(kind)
    if h != d:
        raise ValueError("the oracle-gate construction needs hidden == d")
    H = hadamard(d)
    w1 = H * 2.0 ** -GATE_SHIFT
    w2 = round_bf16(gate @ H.T * (2.0 ** (GATE_SHIFT + 1) / d))
    return pb.PredictorModel("arch2", w1, np.zeros(h), w2, np.zeros(E), dropout_rate=0.0)


def make_layer(kind: str, d: int, h: int, E: int, k: int, n: int, seed: int, device):
    """(model, x bf16 [n, d] on device, truth int32 [n, k] ascending on device)."""
    import torch
    gate = gate_weights(E, d, 10_000 + seed)
    model = make_predictor(kind, d, h, E, seed, gate)
    g = torch.Generator(device=device)
    g.manual_seed(20_000 + seed)
    x = torch.empty((n, d), dtype=torch.bfloat16, device=device)
    gt = torch.as_tensor(gate, dtype=torch.float32, device=device)
    truth = torch.empty((n, k), dtype=torch.int32, device=device)
    step = 1 << 18
    for s in range(0, n, step):
        xf = torch.randn((min(step, n - s), d), device=device, generator=g, dtype=torch.float32)
        xf = (xf - xf.mean(1, keepdim=True)) * torch.rsqrt(xf.var(1, unbiased=False, keepdim=True) + 1e-5)
        xb = xf.to(torch.bfloat16)
        x[s: s + xb.shape[0]] = xb
        xf = xb.float()
        xn = (xf - xf.mean(1, keepdim=True)) * torch.rsqrt(xf.var(1, unbiased=False, keepdim=True) + 1e-5)
        truth[s: s + xb.shape[0]] = torch.topk(xn @ gt.T, k, dim=1).indices.sort(dim=1).values.to(torch.int32)
    return model, x, truth
