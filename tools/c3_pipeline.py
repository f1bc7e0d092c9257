"""BASELINE configs[2]: Qwen3-30B-A3B shape (d=2048, E=128, top-8, 48 layers),
predictor inference + expert prefetch overlapped with attention.

Per layer and decode batch B: on the main stream the pre-attention predictor
(fused K1 + fix-up on the batch's normalised hidden states) then the layer's
attention (decode GQA stand-in: 32 query heads over 4 KV heads, head_dim 128,
4096 cached bf16 tokens per sequence, as grouped batched matmuls + softmax so
the KV cache is read once); on a side stream, as soon as the predictor finishes, the prefetch of
the predicted experts (K8 plan + copy engines, Qwen3 expert = 3*2048*768*2 B)
into a device cache. Reported per layer: predictor / attention / load times,
and the stall max(0, load_end - attention_end) (pipesim.py:281-285)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
from paper_2511_10676_b200 import prefetch as pf  # noqa: E402
from oracle import oracle as O  # noqa: E402

D, H, E, K, L = 2048, 2048, 128, 8, 48
dev = torch.device("cuda")
layers = []
for li in range(4):  # 4 distinct predictors cycled over the 48 layers (weights are L2-sized anyway)
    m = pb.init_model("arch2", D, H, E, seed=li)
    m.w1, m.w2 = O.round_bf16(m.w1), O.round_bf16(m.w2)
    layers.append(m.to_device())
store = pf.ExpertStore(E, pf.QWEN3_EXPERT_BYTES)
cache = pf.ExpertCache(E, pf.QWEN3_EXPERT_BYTES, E)
p = pf.Prefetcher(store, cache)
peak = pf.measure_h2d_peak(1 << 30, 5)
T_CTX = 4096


def attention(qg, k, v):
    """Decode GQA: qg [B, 4, 8, 128], k/v [B, 4, T, 128] -> [B, 4, 8, 128]."""
    s = torch.matmul(qg, k.transpose(-1, -2)) * (128 ** -0.5)
    return torch.matmul(torch.softmax(s.float(), dim=-1).to(qg.dtype), v)
main = torch.cuda.current_stream()
out = {"config": "Qwen3-30B-A3B shape, 48 layers, decode", "h2d_peak_gbs": peak,
       "expert_bytes": pf.QWEN3_EXPERT_BYTES, "batches": []}
for B in (1, 8, 32, 128, 256):
    x = torch.randn((B, D), device=dev).to(torch.bfloat16)
    qb = torch.randn(B, 4, 8, 128, device=dev, dtype=torch.bfloat16)
    kb = torch.randn(B, 4, T_CTX, 128, device=dev, dtype=torch.bfloat16)
    vb = torch.randn(B, 4, T_CTX, 128, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        attention(qb, kb, vb)
        layers[0].topk(x, K, validate=False)
    torch.cuda.synchronize()
    for mode in ("copy_engine", "sm_gather_16cta"):
        rows = []
        for li in range(L):
            cache.reset()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record(main)
            ids = layers[li % 4].topk(x, K, validate=False)  # predictor on the attention input (no host sync)
            ev[1].record(main)
            if mode == "sm_gather_16cta":
                # GPU-driven plan + gather on 16 CTAs; the remaining SMs run the attention
                p.copy.wait_event(ev[1])
                p.load_sm_gather(ids, 16)
                attention(qb, kb, vb)
                ev[2].record(main)
            else:
                # attention is enqueued first; the host then reads the (tiny) plan,
                # which waits only for the predictor, and issues one copy per expert
                attention(qb, kb, vb)
                ev[2].record(main)
                p.copy.wait_event(ev[1])
                p.load_copy_engine(ids)
            ev[3].record(p.copy)
            torch.cuda.synchronize()
            t_pred = ev[0].elapsed_time(ev[1])
            t_attn_end = ev[0].elapsed_time(ev[2])
            t_load_end = ev[0].elapsed_time(ev[3])
            n = int(p.need_count.item())
            rows.append((t_pred, t_attn_end - t_pred, t_load_end - t_pred, max(0.0, t_load_end - t_attn_end), n))
        r = np.array(rows)
        out["batches"].append({"batch": B, "mode": mode, "predict_ms": float(r[:, 0].mean()),
                               "attention_ms": float(r[:, 1].mean()), "load_ms": float(r[:, 2].mean()),
                               "stall_ms": float(r[:, 3].mean()), "experts_loaded": float(r[:, 4].mean()),
                               "load_gbs": float(r[:, 4].mean() * pf.QWEN3_EXPERT_BYTES / (r[:, 2].mean() / 1e3) / 1e9)})
    # attention alone (no concurrent load) for reference
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(main)
    for _ in range(10):
        attention(qb, kb, vb)
    a1.record(main)
    torch.cuda.synchronize()
    out["batches"].append({"batch": B, "mode": "attention_alone", "attention_ms": a0.elapsed_time(a1) / 10})
print(json.dumps(out))
