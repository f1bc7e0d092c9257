"""Predictor latency per decode batch: exact fp64 decode kernel vs the
tensor-core path (K1 + fix-up), Qwen3 and DSV2L shapes, CUDA-event timed over
200 back-to-back calls (no host sync inside)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
from oracle import oracle as O  # noqa: E402

res = []
for name, E, k in (("qwen3", 128, 8), ("dsv2l", 64, 6)):
    m = pb.init_model("arch2", 2048, 2048, E, seed=1)
    m.w1, m.w2 = O.round_bf16(m.w1), O.round_bf16(m.w2)
    dev = m.to_device()
    for n in (1, 2, 4, 8, 16, 32, 64, 128, 256, 1024, 4096, 16384, 65536):
        x = torch.randn((n, 2048), device="cuda").to(torch.bfloat16)
        row = {"shape": name, "batch": n}
        for path, lim in (("decode_fp64", 1 << 30), ("tensor_k1", 0)):
            if path == "decode_fp64" and n > 256:
                continue
            flop = 2 * n * (2048 * 2048 + 2048 * E)
            dev.decode_max_tokens = lim
            for _ in range(10):
                dev.topk(x, k, validate=False)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(200):
                dev.topk(x, k, validate=False)
            b.record()
            torch.cuda.synchronize()
            row[path + "_eager_us"] = a.elapsed_time(b) / 200 * 1e3
            # device time: 20 calls captured in one CUDA graph (no host launch cost)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                for _ in range(3):
                    dev.topk(x, k, validate=False)
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    dev.topk(x, k, validate=False)
            g.replay()
            torch.cuda.synchronize()
            a.record()
            for _ in range(10):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            row[path + "_graph_us"] = a.elapsed_time(b) / 200 * 1e3
            row[path + "_tflops"] = flop / (row[path + "_graph_us"] * 1e-6) / 1e12
        res.append(row)
        print(json.dumps(row), flush=True)
