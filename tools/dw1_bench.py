"""Timing of the tcgen05 dW1 GEMM (moep_dw1_bf16) at the Phi training shape
(16,384 tokens, h = 2048, d = 4096) for both passes, against cuBLAS on the
same operands (torch.mm), CUDA events, median of 20."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_10676_b200._lib import check, lib, ptr  # noqa: E402

n, h, d = 16384, 2048, 4096
for passes in (1, 2):
    da = torch.randn((n, passes * h), device="cuda").to(torch.bfloat16)
    x = torch.randn((n, d), device="cuda").to(torch.bfloat16)
    out = torch.empty((h, d), dtype=torch.float32, device="cuda")
    need = int(lib().moep_dw1_workspace_floats(h, d, n, passes))
    ws = torch.zeros(max(need, 1), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def ours():
        check(lib().moep_dw1_bf16(ptr(da), ptr(x), n, h, d, passes, ptr(out), ptr(ws), need, st), "dw1")

    def cublas():
        c = torch.mm(da.t(), x, out_dtype=torch.float32)
        if passes == 2:
            torch.add(c[:h], c[h:], out=out)

    res = {}
    for name, fn in (("ours", ours), ("cublas", cublas)):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        res[name] = {"ms": ms, "tflops": 2.0 * passes * n * h * d / ms / 1e9}
    print(json.dumps({"passes": passes, "splits_workspace_floats": need, **res}))
