"""K0 timing: 1M x d bf16 rows, rmsnorm(gamma) and layernorm(gamma, beta) ->
bf16 x_hat. 4 bytes per element of algorithmic traffic (read x, write x_hat)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_10676_b200.engine import input_norm  # noqa: E402

n = 1 << 20
for d in (2048, 4096):
    x = (torch.randn((n, d), device="cuda") * 2).to(torch.bfloat16)
    gamma = np.random.default_rng(0).uniform(0.5, 1.5, d)
    beta = 0.1 * np.random.default_rng(1).standard_normal(d)
    st = torch.zeros(2, dtype=torch.int32, device="cuda")
    for kind, b in (("rmsnorm", None), ("layernorm", beta)):
        for _ in range(3):
            input_norm(x, kind, gamma, b, status=st)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            input_norm(x, kind, gamma, b, status=st)
        e.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(e) / 10
        print(json.dumps({"d": d, "kind": kind, "rows": n, "ms": ms, "gbs": 4 * n * d / ms / 1e6, "exact_warps": int(st[1])}))
