"""Achieved bandwidth of the HBM-bound helper kernels against the measured HBM
peak (MEASURED_PEAKS.json), each timed alone with CUDA events (best of 10,
inputs larger than L2 where the shape allows), algorithmic bytes as DESIGN §4
states them:

  K7  moep_eval_logits   (fp32 logits [N, E] + int32 truth [N, k]) -> counters
  K7  moep_topk_logits   fp32 logits [N, E] -> int32 ids [N, m]
  K0  moep_input_norm    bf16 x [N, d] -> bf16 x_hat [N, d] (layernorm, fp64 stats)
  K3  moep_labels        fp32 scores [N, E] -> int32 rank + u8 mask [N, E], int32 pairs [N]
  K4  moep_loss+finalize fp32 logits/scores [N, E], int32 rank, u8 mask -> fp32 dz [N, E] (+ hinge)

    python tools/kernel_rooflines.py [--out profiles/r01_kernel_rooflines.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2511_10676_b200 as pb  # noqa: E402
from paper_2511_10676_b200 import losses  # noqa: E402
from paper_2511_10676_b200.engine import eval_logits_device, topk_logits_device  # noqa: E402


def best_ms(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda")
    _, _, hbm, src = bench.peaks()
    res = {"hbm_peak_gbs": hbm, "peak_source": src, "kernels": []}

    def add(name, ms, nbytes, note):
        gbs = nbytes / (ms / 1e3) / 1e9
        res["kernels"].append({"kernel": name, "ms": ms, "algorithmic_bytes": nbytes, "gbs": gbs,
                               "frac_of_hbm": gbs / hbm, "shape": note})
        print(f"{name:28s} {ms:8.3f} ms  {gbs:8.1f} GB/s  {gbs / hbm * 100:5.1f} %  {note}", flush=True)

    g = torch.Generator(device=dev).manual_seed(0)
    # K7 over DSV2L-shaped logits (4 M tokens: 1 GiB of fp32 logits, > L2)
    n, e, k = 1 << 22, 64, 6
    z = torch.randn((n, e), device=dev, generator=g)
    truth = torch.argsort(torch.rand((n, e), device=dev, generator=g), dim=1)[:, :k].sort(dim=1).values.int()
    ms = best_ms(lambda: eval_logits_device(z, truth, k, e, [6, 10, 64]))
    add("K7 eval_logits", ms, n * (4 * e + 4 * k), f"N={n}, E={e}, k={k}, M=[6,10,64]")
    ms = best_ms(lambda: topk_logits_device(z, 6))
    add("K7 topk_logits", ms, n * (4 * e + 4 * 6), f"N={n}, E={e}, m=6")
    del z, truth
    # K0 input norm (layernorm with affine, bf16 in/out): 1 M tokens x 2048 (4 GiB in + 4 GiB out)
    m = pb.init_model("arch2", 2048, 2048, 64, seed=0)
    dp = m.to_device()
    nx, d = 1 << 20, 2048
    x = torch.randn((nx, d), device=dev, generator=g).to(torch.bfloat16)
    gam = np.ones(d)
    bet = np.zeros(d)
    ms = best_ms(lambda: dp.normalize(x, "layernorm", gam, bet))
    add("K0 input_norm (layernorm)", ms, nx * d * 4, f"N={nx}, d={d}, bf16 -> bf16")
    del x
    # K3 labels + K4 ranking loss at the Phi shape, 4 M tokens x 16 experts
    nl, el = 1 << 22, 16
    s = torch.softmax(torch.randn((nl, el), device=dev, generator=g), dim=1).float().contiguous()
    ms = best_ms(lambda: losses.BatchLabels.from_scores(s, 2))
    add("K3 labels", ms, nl * (4 * el + 4 * el + el + 4), f"N={nl}, E={el}, k=2")
    lab = losses.BatchLabels.from_scores(s, 2)
    sc, mask, rank = lab.to_device(torch.float32, dev)
    zl = torch.randn((nl, el), device=dev, generator=g).contiguous()
    spec = losses.LossSpec("ranking")
    ms = best_ms(lambda: losses.device_loss(spec, zl, sc, mask, rank))
    # read z, s, rank, mask; write dz and the hinge gradient; finalize re-reads both, writes dz
    add("K4 ranking loss + finalize", ms, nl * el * (4 + 4 + 4 + 1 + 4 + 4 + 4 + 4 + 4), f"N={nl}, E={el}")
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
