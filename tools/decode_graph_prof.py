"""Kernels of one captured pre-attention decode step (Qwen3 shape, B = 1 / 8):
ncu --metrics gpu__time_duration.sum python tools/decode_graph_prof.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2511_10676_b200.deploy import HookPointPredictor  # noqa: E402

D, E3 = 2048, 128
H_ = W.hadamard(D)
gate = W.gate_weights(E3, D, 30_000)
m = pb.PredictorModel("arch2", H_ * 2.0 ** -W.GATE_SHIFT, np.zeros(D),
                      W.round_bf16(gate @ H_.T * (2.0 ** (W.GATE_SHIFT + 1) / D)), np.zeros(E3), dropout_rate=0.0)
hp = HookPointPredictor(m, 8, "rmsnorm", np.ones(D))
for B in (1, 8):
    hid = torch.randn((B, D), device="cuda").to(torch.bfloat16)
    gh = hp.graph(B)
    for _ in range(3):
        gh.pre_attention(hid, prefetch=False)
    torch.cuda.synchronize()
print("ok")

# timing without a profiler: eager vs graph replay, CUDA events, median of 50
import statistics  # noqa: E402
for B in (1, 8, 32):
    hid = torch.randn((B, D), device="cuda").to(torch.bfloat16)
    gh = hp.graph(B)
    res = {}
    for name, fn in (("eager", lambda: hp.pre_attention(hid, prefetch=False)),
                     ("graph", lambda: gh.pre_attention(hid, prefetch=False))):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(50):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res[name] = round(statistics.median(ts), 1)
    print("B", B, "us", res)
