"""Where K1's logit error comes from (DSV2L shape, 16k tokens): total error of
the fp32 logits vs the fp64 oracle, and the part already present in the
GEMM1 pre-activations (a_out, fp32 from the tensor core) pushed through an
exact fp64 activation + GEMM2. The difference is the epilogue's fp32
activation, the bf16 hi/lo split and GEMM2's fp32 TMEM accumulation.
Ratios are |dz| / (||h||_2 * max_e ||w2_e||_2), the scale the K1 margin uses."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
from oracle import oracle as O  # noqa: E402  (measurement tool: the oracle is the checker)

import workloads as W  # noqa: E402

n, d, h, e = 16384, 2048, 2048, 64
KIND = sys.argv[1] if len(sys.argv) > 1 else "random"
m, xt0, _ = W.make_layer(KIND, d, h, e, 6, n, seed=5, device="cuda")
x = xt0.double().cpu().numpy()
print("workload", KIND)
p = {"arch": "arch2", "w1": m.w1, "b1": m.b1, "w2": m.w2, "b2": m.b2}
zref, cache = O.forward_eval(p, x)
dev = m.to_device()
lg = torch.empty((n, e), dtype=torch.float32, device="cuda")
a_out = torch.empty((n, h), dtype=torch.float32, device="cuda")
xb = torch.from_numpy(x).to("cuda", torch.bfloat16)
orig = dev._k1
flags, _, _ = dev._k1(xb, logits=lg)
# pre-activations from the training forward path of the same kernel (a_out)
from paper_2511_10676_b200 import _lib  # noqa: E402
A = _lib.PredictArgs()
A.n_tokens, A.d, A.hidden, A.n_experts, A.arch = n, d, h, e, dev.arch_code
A.x, A.w1, A.w2, A.b1, A.b2 = xb.data_ptr(), dev.w1_bf16.data_ptr(), dev.w2_bf16.data_ptr(), dev.b1_f32.data_ptr(), dev.b2_f32.data_ptr()
A.tau_abs, A.tau_rel, A.w2_norm = dev.tau_abs, dev.tau_rel, dev.w2_norm
fl = torch.empty(n, dtype=torch.uint8, device="cuda"); fli = torch.empty(n, dtype=torch.int32, device="cuda")
fc = torch.zeros(1, dtype=torch.int32, device="cuda")
A.flags, A.flag_list, A.flag_count, A.a_out = fl.data_ptr(), fli.data_ptr(), fc.data_ptr(), a_out.data_ptr()
A.logits = lg.data_ptr()
_lib.check(_lib.lib().moep_predict_bf16(A, torch.cuda.current_stream().cuda_stream), "k1")
torch.cuda.synchronize()
scale = np.linalg.norm(cache["h"], axis=1) * np.linalg.norm(m.w2, axis=1).max()
tot = np.abs(lg.double().cpu().numpy() - zref).max(axis=1) / scale
a64 = a_out.double().cpu().numpy()
z_g1 = O.silu(a64) @ m.w2.T + m.b2
g1 = np.abs(z_g1 - zref).max(axis=1) / scale
print(f"total     : max {tot.max():.3e}  p99.9 {np.quantile(tot, 0.999):.3e}  mean {tot.mean():.3e}")
print(f"GEMM1 only: max {g1.max():.3e}  p99.9 {np.quantile(g1, 0.999):.3e}  mean {g1.mean():.3e}")
# emulate the hi/lo split exactly on the GPU's pre-activations with fp64 silu
hh = O.silu(a64)
hi = O.round_bf16(hh)
lo = O.round_bf16(hh - hi)
z_split = (hi + lo) @ m.w2.T + m.b2
sp = np.abs(z_split - zref).max(axis=1) / scale
print(f"GEMM1+split (exact act, exact GEMM2): max {sp.max():.3e}  mean {sp.mean():.3e}")
print(f"flagged: {int(fc.item())} of {n} at tau_rel {dev.tau_rel}")
