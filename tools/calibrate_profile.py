"""Measured B200 HardwareProfile for the reference's pipeline simulator
(pkg/src/moepredict/pipesim.py:33-105, schema of
HardwareProfile.to_json). One DeepSeek-V2-Lite-shaped decoder layer at a
decode batch of 1 token, every stage timed with CUDA events (median of 50):

  t_pre_norm      K0 RMSNorm of the layer input (d = 2048)
  t_attn          decode attention stand-in: 16 heads x 4096 cached tokens, head_dim 128 (SDPA)
  t_post_norm     K0 RMSNorm after attention
  t_select        the layer's own router: x . W_g^T (64 x 2048) + exact top-6 (K7)
  t_expert_compute 6 SwiGLU experts (2048 -> 1408 -> 2048, bf16)
  t_load_mem_per_expert  one 17,301,504 B expert, pinned host -> device (copy engine)
  t_load_disk_per_expert one expert read from a local file (page cache) into pinned memory
  t_predict       this repo's pre-attention predictor for 1 token (exact decode kernel)
  parallel_load_slots 1 (one copy engine per direction is used)

Writes the JSON to argv[1] (default profiles/r01_b200_hardware_profile.json).
The file loads with the reference's HardwareProfile.from_json (same keys).
"""
import json
import os
import statistics
import sys
import tempfile
import time

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
from paper_2511_10676_b200 import prefetch as pf  # noqa: E402
from paper_2511_10676_b200.engine import topk_logits_device  # noqa: E402
from oracle import oracle as O  # noqa: E402  (bf16 rounding of the random weights only)

out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r01_b200_hardware_profile.json")
dev = torch.device("cuda")
D, E, K, FF = 2048, 64, 6, 1408


def timed(fn, reps=50):
    ts = []
    for _ in range(5):
        fn()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), statistics.pstdev(ts)


m = pb.init_model("arch2", D, D, E, seed=0)
m.w1, m.w2 = O.round_bf16(m.w1), O.round_bf16(m.w2)
dp = m.to_device()
x = torch.randn((1, D), device=dev)
gamma = torch.ones(D, dtype=torch.float64, device=dev)
q = torch.randn(1, 16, 1, 128, device=dev, dtype=torch.bfloat16)
kv = torch.randn(1, 16, 4096, 128, device=dev, dtype=torch.bfloat16)
wg = torch.randn((E, D), device=dev, dtype=torch.bfloat16) / D ** 0.5
experts = [[torch.randn(FF, D, device=dev, dtype=torch.bfloat16) / D ** 0.5 for _ in range(3)] for _ in range(K)]
xb = x.to(torch.bfloat16)


def swiglu():
    y = torch.zeros_like(xb)
    for w_gate, w_up, w_down in experts:
        h = F.silu(xb @ w_gate.T) * (xb @ w_up.T)
        y = y + h @ w_down  # w_down stored [FF, D]
    return y


res, std = {}, {}
res["t_pre_norm"], std["t_pre_norm"] = timed(lambda: dp.normalize(x, "rmsnorm", gamma))
res["t_attn"], std["t_attn"] = timed(lambda: F.scaled_dot_product_attention(q, kv, kv))
res["t_post_norm"], std["t_post_norm"] = timed(lambda: dp.normalize(x, "rmsnorm", gamma))
res["t_select"], std["t_select"] = timed(lambda: topk_logits_device((xb @ wg.T).float(), K))
res["t_expert_compute"], std["t_expert_compute"] = timed(swiglu)
res["t_predict"], std["t_predict"] = timed(lambda: dp.topk(xb, K, validate=False))

store = pf.ExpertStore(2, pf.DSV2L_EXPERT_BYTES)
dst = torch.empty(pf.DSV2L_EXPERT_BYTES, dtype=torch.uint8, device=dev)
res["t_load_mem_per_expert"], std["t_load_mem_per_expert"] = timed(
    lambda: dst.copy_(store.blob(0), non_blocking=True), reps=20)

# "disk": one expert blob read from a local file into pinned memory (page cache; cold
# disk reads are not reproducible in this sandbox)
blob = store.blob(1).numpy()
fd, path = tempfile.mkstemp()
os.write(fd, blob.tobytes())
os.close(fd)
pinned = torch.empty(pf.DSV2L_EXPERT_BYTES, dtype=torch.uint8).pin_memory()
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    with open(path, "rb", buffering=0) as f:
        f.readinto(memoryview(pinned.numpy()))
    ts.append((time.perf_counter() - t0) * 1e3)
os.remove(path)
res["t_load_disk_per_expert"] = statistics.median(ts)
std["t_load_disk_per_expert"] = statistics.pstdev(ts)

profile = {"name": "b200_measured", **{k: float(v) for k, v in res.items()}, "parallel_load_slots": 1,
           "std": {k: float(v) for k, v in std.items()}}
order = ["name", "t_pre_norm", "t_attn", "t_post_norm", "t_select", "t_expert_compute", "t_load_disk_per_expert",
         "t_load_mem_per_expert", "t_predict", "parallel_load_slots", "std"]
with open(out_path, "w") as f:
    json.dump({k: profile[k] for k in order}, f, indent=2)
    f.write("\n")
print(json.dumps(profile))
