"""Training-step throughput at the Phi-mini shape (BASELINE configs[3]):
d=4096, h=2048, E=16, k=2, arch2 + ranking-aware loss, Adam, fp32 tensor-core
mode; one step = forward (K1) + K4 loss + K5 + dW1 GEMM + K6 over a global
batch of `--batch` synthetic tokens. Also times the oracle (numpy fp64) step at
N=256 on the host for reference, and checks one step against it."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
from oracle import oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=4096)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--k1-kernel", type=int, default=0, help="forced forward K1 kernel (moep_predict_args.kernel)")
args = ap.parse_args()
d, h, e, k, n = 4096, 2048, 16, 2, args.batch
rng = np.random.default_rng(0)
m = pb.init_model("arch2", d, h, e, seed=1)
m.w1, m.w2 = O.round_bf16(m.w1), O.round_bf16(m.w2)
dev = torch.device("cuda")
x = torch.randn((n, d), device=dev).to(torch.bfloat16)
gate = torch.randn((e, d), device=dev) / 64.0
scores = torch.softmax(x.float() @ gate.T, dim=1).double()
lab = pb.BatchLabels.from_scores(scores, k)
dt = torch.float32 if args.precision in ("fp32", "bf16") else torch.float64
s_, mk, rk = lab.true_scores.to(dt).contiguous(), lab.topk_mask.to(torch.uint8).contiguous(), lab.rank_of.contiguous()
tr = pb.DeviceTrainer(m, pb.LossSpec(family="ranking"), "adam", 1e-3, precision=args.precision)
tr.k1_kernel = args.k1_kernel
xin = x if args.precision in ("fp32", "bf16") else x.double()
for _ in range(3):
    tr.step(xin, s_, mk, rk)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(args.steps):
    out = tr.step(xin, s_, mk, rk)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / args.steps
flop = (4 * d * h + 6 * h * e) * n
# CPU oracle step at N=256 (reference default batch)
p = O.init_params("arch2", d, h, e, seed=1)
xs = O.round_bf16(rng.standard_normal((256, d)))
sc = O.softmax(rng.standard_normal((256, e)), axis=1)
olab = O.batch_labels(sc, k)
st, t0 = {}, time.perf_counter()
for t in range(3):
    z, cache = O.forward_eval(p, xs)
    lv, dz = O.loss_and_grad({"family": "ranking"}, z, olab)
    g = O.backward_eval(p, cache, dz)
    O.adam_step(p, {kk: g[kk] for kk in ("w1", "b1", "w2", "b2")}, st, t + 1)
cpu_s = (time.perf_counter() - t0) / 3
print(json.dumps({"workload": "Phi-mini shape arch2+ranking Adam training step", "precision": args.precision,
                  "batch_tokens": n, "ms_per_step": ms, "tokens_per_s": n / (ms / 1e3),
                  "tflops_algorithmic": flop / (ms / 1e3) / 1e12, "flop_per_token": 4 * d * h + 6 * h * e,
                  "roofline_tokens_per_s_sustained": 1366.2e12 / (4 * d * h + 6 * h * e),
                  "loss": float(out[0].item()),
                  "cpu_oracle_step_n256_s": cpu_s, "cpu_oracle_tokens_per_s": 256 / cpu_s,
                  "cpu_cores": os.cpu_count()}))
