"""Throughput of the GPU synthetic teacher (K11).

DSV2L-shaped teacher (d=2048, E=64, top-6, identity transform + layer norm,
optional noise row): generate_dataset_device over N samples, timed with CUDA
events (best of R), plus the normals kernel alone and its write bandwidth
(12 B per normal: fp64 + fp32 copies). CPU reference: the reference's own
per-sample loop (synthgen.py:170-174: numpy Generator(Philox(key)) per sample)
+ layer_norm + gate softmax on a bounded sample, timed on the host.

    python tools/synthgen_bench.py [--n 1048576] [--noise 0.1] [--out profiles/r01_synthgen.json]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_10676_b200 import synthgen as sg  # noqa: E402
from paper_2511_10676_b200._lib import check, lib, ptr  # noqa: E402


def cpu_reference(gate, n, d, noise, seed):
    t0 = time.perf_counter()
    x = np.empty((n, d))
    nz = np.empty((n, d)) if noise > 0 else None
    for i in range(n):
        g = np.random.Generator(np.random.Philox(key=((seed & 0xFFFFFFFFFFFFFFFF) << 64) + i))
        x[i] = g.standard_normal(d)
        if nz is not None:
            nz[i] = g.standard_normal(d)
    post = x.copy()
    if nz is not None:
        post += noise * nz
    post = (post - post.mean(-1, keepdims=True)) / np.sqrt(post.var(-1, keepdims=True) + 1e-5)
    z = post @ gate.T
    z = z - z.max(-1, keepdims=True)
    e = np.exp(z)
    s = (e / e.sum(-1, keepdims=True)).astype(np.float32)
    np.sort(np.argsort(-s.astype(np.float64), axis=1, kind="stable")[:, :6], axis=1)
    return n / (time.perf_counter() - t0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--noise", type=float, default=0.0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu-n", type=int, default=4096)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    d, e, k, seed = 2048, 64, 6, 0
    gate = np.random.default_rng(0).standard_normal((e, d)) / np.sqrt(d)
    t = sg.TeacherSpec(sg.RouterSpec(d, e, k, gate), noise_sigma=a.noise, seed=seed)
    sg.generate_dataset_device(t, 4096)  # warm-up
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(a.reps):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        dt = sg.generate_dataset_device(t, a.n)
        s1.record()
        torch.cuda.synchronize()
        best = min(best, s0.elapsed_time(s1))
        del dt
    # normals kernel alone (fp64 + fp32 rows, the noise row when enabled)
    m = min(a.n, 1 << 18)
    x64 = torch.empty((m, d), dtype=torch.float64, device="cuda")
    x32 = torch.empty((m, d), dtype=torch.float32, device="cuda")
    nz = torch.empty((m, d), dtype=torch.float64, device="cuda") if a.noise > 0 else None
    st = torch.cuda.current_stream().cuda_stream
    kbest = 1e30
    for _ in range(a.reps + 1):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        check(lib().moep_teacher_normals(seed, 0, m, d, int(a.noise > 0), ptr(x64), ptr(x32), ptr(nz), st), "normals")
        s1.record()
        torch.cuda.synchronize()
        kbest = min(kbest, s0.elapsed_time(s1))
    normals = m * d * (2 if a.noise > 0 else 1)
    bytes_w = m * d * 12 + (m * d * 8 if a.noise > 0 else 0)
    # stage breakdown of one 262144-sample chunk (the default chunk of generate_dataset_device)
    c = min(a.n, 262144)
    tt = sg._Teacher(t, torch.device("cuda"))
    acts = torch.empty((c, d), dtype=torch.float32, device="cuda")
    sc = torch.empty((c, e), dtype=torch.float32, device="cuda")
    tk = torch.empty((c, k), dtype=torch.int32, device="cuda")
    x64c = torch.empty((c, d), dtype=torch.float64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for rep in range(2):
        ev[0].record()
        check(lib().moep_teacher_normals(seed, 0, c, d, 0, ptr(x64c), ptr(acts), None, st), "normals")
        ev[1].record()
        check(lib().moep_layer_norm_np(ptr(x64c), c, d, 1e-5, ptr(x64c), st), "ln")
        ev[2].record()
        logits = tt._gemm(x64c, tt.gate)  # moep_dgemm_nt (fp64 tensor cores)
        ev[3].record()
        check(lib().moep_teacher_finish(ptr(logits), c, e, k, ptr(sc), ptr(tk), st), "finish")
        ev[4].record()
        torch.cuda.synchronize()
    stages = {n: ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(["normals", "layer_norm", "gate_gemm", "finish"])}
    cpu = cpu_reference(gate, a.cpu_n, d, a.noise, seed)
    res = {"workload": "DSV2L-shaped teacher (d=2048, E=64, top-6, identity + layer_norm"
                       + (f", noise {a.noise}" if a.noise > 0 else "") + ")",
           "samples": a.n, "ms": best, "samples_per_s": a.n / (best / 1e3),
           "normals_kernel": {"samples": m, "ms": kbest, "normals_per_s": normals / (kbest / 1e3),
                              "write_gbs": bytes_w / (kbest / 1e3) / 1e9},
           "cpu_reference": {"samples_per_s": cpu, "sample": f"{a.cpu_n} samples, numpy per-sample Philox loop "
                             "(synthgen.py:170-174) + layer_norm + gate softmax + top-k", "cores": os.cpu_count()},
           "speedup_vs_cpu": a.n / (best / 1e3) / cpu,
           "stages_ms_per_chunk": stages, "chunk": c}
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
