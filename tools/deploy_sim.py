"""Deployment at the hook point, measured: the predictor
runs on the pre-attention normalised hidden state of each MoE layer
(hooks.py:19, 113-114: the exporter's `input_layernorm` hook), its predicted
experts are prefetched while the attention runs, and experts the router then
selects but the prediction missed are loaded on demand ("emergency" loads) —
the prefetch_hit / prefetch_miss schedules that pipesim.py:272-305 only
models, here executed on the B200 with real copies.

DSV2L-shaped stack (d = 2048, 64 experts of 17,301,504 B, top-6), decode
batch 1, 26 layers x `steps` tokens. Per layer:
  x_hat = RMSNorm(x)                                   (K0)
  predicted = top-m(predictor(x_hat))                  (decode kernel, no host sync)
  [prefetch] copy engines load predicted - resident    (side stream)
  attention stand-in (SDPA, 16 heads x 4096 cached tokens)
  router: top-6 of W_g . RMSNorm(x + attention mix)    (the true experts)
  emergency loads of true - loaded                     (copy engines)
  6 SwiGLU experts computed from the cache slots
The predictor is the oracle-gate construction of the reference's metric tests
(test_metrics.py:185-192: w1 = eps*I, w2 = 2*W_g/eps), so its top-m agrees with
the router up to the attention mix (`--mix` sets how much the residual stream
moves between the predictor's and the router's input).
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
from paper_2511_10676_b200 import prefetch as pf  # noqa: E402
from paper_2511_10676_b200.engine import topk_logits_device  # noqa: E402
from oracle import oracle as O  # noqa: E402  (bf16 rounding of the constructed weights only)

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=26)
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--mix", type=float, default=0.3)
ap.add_argument("--m", type=int, default=6, help="prefetch set size (6 = k, 10 = over-provisioned)")
args = ap.parse_args()

D, E, K, FF = 2048, 64, 6, 1408
dev = torch.device("cuda")
rng = np.random.default_rng(0)
L = args.layers
eps = 2.0 ** -6
gates, preds = [], []
for layer in range(min(L, 4)):  # 4 distinct layers cycled (weights are per layer in a real model)
    wg = rng.standard_normal((E, D)) / np.sqrt(D)
    m = pb.PredictorModel("arch2", O.round_bf16(eps * np.eye(D)), np.zeros(D), O.round_bf16(2.0 * wg / eps),
                          np.zeros(E))
    preds.append(m.to_device())
    gates.append(torch.from_numpy(wg).to(dev, torch.bfloat16))
gamma = torch.ones(D, dtype=torch.float64, device=dev)
q = torch.randn(1, 16, 1, 128, device=dev, dtype=torch.bfloat16)
kv = torch.randn(1, 16, 4096, 128, device=dev, dtype=torch.bfloat16)
store = pf.ExpertStore(E, pf.DSV2L_EXPERT_BYTES)
cache = pf.ExpertCache(E, pf.DSV2L_EXPERT_BYTES, E, device=dev)
p = pf.Prefetcher(store, cache)
main = torch.cuda.current_stream()


def expert_compute(xb, slots):
    """6 SwiGLU experts; each cache slot holds [gate | up | down] bf16 [1408, 2048]."""
    y = torch.zeros_like(xb)
    for s in slots:
        w = cache.slot(s).view(torch.bfloat16)[: 3 * FF * D].view(3, FF, D)
        y = y + (F.silu(xb @ w[0].T) * (xb @ w[1].T)) @ w[2]
    return y


def run(mode):
    lat, misses, loaded = [], [], []
    for step in range(args.steps):
        for layer in range(L):
            li = layer % len(preds)
            x = torch.randn((1, D), device=dev)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(main)
            xh = preds[li].normalize(x, "rmsnorm", gamma)
            n_pref = 0
            slot_host = {}
            next_free = 0
            if mode == "prefetch":
                ids = preds[li].topk(xh, args.m, validate=False)
                pred_done = torch.cuda.Event()
                pred_done.record(main)
            F.scaled_dot_product_attention(q, kv, kv)          # this layer's attention (the window)
            if mode == "prefetch":
                p.copy.wait_event(pred_done)
                n_pref = p.load_copy_engine(ids)                # host reads the plan (waits for the predictor only)
                for e, sl in zip(p.h_plan[:n_pref].tolist(), p.h_plan[E:E + n_pref].tolist()):
                    slot_host[e] = sl
                next_free = n_pref
            x2 = x + args.mix * torch.randn_like(x)            # residual stream after attention
            xh2 = preds[li].normalize(x2, "rmsnorm", gamma).to(torch.bfloat16)
            true = topk_logits_device((xh2 @ gates[li].T).float(), K)[0].tolist()   # router (host sync)
            miss = [e for e in true if e not in slot_host]
            main.wait_stream(p.copy)                           # prefetched experts landed
            for e in miss:                                      # emergency loads (copy engine)
                slot_host[e] = next_free
                cache.slot(next_free).copy_(store.blob(e), non_blocking=True)
                next_free += 1
            expert_compute(xh2, [slot_host[e] for e in true])
            ev1.record(main)
            torch.cuda.synchronize()
            lat.append(ev0.elapsed_time(ev1))
            misses.append(len(miss))
            loaded.append(n_pref + len(miss))
    return {"mode": mode, "layer_ms_mean": statistics.mean(lat), "layer_ms_p50": statistics.median(lat),
            "misses_per_layer": statistics.mean(misses), "experts_loaded_per_layer": statistics.mean(loaded),
            "hit_layers_frac": sum(1 for x in misses if x == 0) / len(misses)}


run("no_prefetch")  # warm up
res = [run("no_prefetch"), run("prefetch")]
out = {"config": f"DSV2L-shaped stack, {L} layers x {args.steps} decode tokens, prefetch set m={args.m}, "
                  f"attention mix {args.mix}", "results": res,
       "token_ms": {r["mode"]: r["layer_ms_mean"] * L for r in res}}
print(json.dumps(out))
