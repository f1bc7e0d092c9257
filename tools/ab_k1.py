"""A/B timing of K1 builds in one process: the product library and variant
builds (tools/variant_lib.py) are loaded side by side (ctypes RTLD_LOCAL) and
timed round-robin on the same 1M-token DSV2L layer, so clock / power drift
hits every variant alike.

    python tools/ab_k1.py tools/_variants/zlo/libmoep_b200.so [...] [--rounds 6] [--kind gate] [--kernels 4,5]
"""
import argparse
import ctypes as C
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_10676_b200 as pb  # noqa: E402
from paper_2511_10676_b200 import _lib  # noqa: E402
import workloads as W  # noqa: E402


def load(path):
    L = C.CDLL(path)
    for name, args in _lib._SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _lib._RESTYPES.get(name, _lib.i32)
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="*")
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--kind", default="gate")
    ap.add_argument("--E", type=int, default=64)
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--kernels", default="0", help="comma list of moep_predict_args.kernel values (0 = auto)")
    args = ap.parse_args()
    dev = torch.device("cuda")
    kernels = [int(v) for v in args.kernels.split(",")]
    libs = [("product", _lib.lib())] + [(p, load(p)) for p in args.libs]
    libs = [(f"{n} k{kv}", L, kv) for n, L in libs for kv in kernels]
    k = 6 if args.E == 64 else (2 if args.E == 16 else 8)
    model, x, truth = W.make_layer(args.kind, args.d, 2048, args.E, k, args.n, seed=1, device=dev)
    dp = pb.DevicePredictor(model, dev)
    part = torch.empty((dp.n_sms, 2 + 6 + 2 * args.E), dtype=torch.int32, device=dev)
    ms_list = [k, k + 4, args.E]
    res = {n: [] for n, _, _ in libs}
    for r in range(args.rounds):
        for name, L, kv in libs:
            _lib._lib = L
            dp.k1_kernel = kv
            run = lambda: dp._k1(x, m_sel=k, bounds=(1, k, k + 4), ids=torch.empty((x.shape[0], k), dtype=torch.int32,
                                                                                   device=dev),
                                 truth=truth, k=k, m_values=ms_list, partials=part)
            run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.reps):
                run()
            b.record()
            torch.cuda.synchronize()
            res[name].append(a.elapsed_time(b) / args.reps)
    for name, v in res.items():
        print(f"{name[-40:]:40s} median {statistics.median(v):.3f} ms  min {min(v):.3f}  all {[round(t, 3) for t in v]}")


if __name__ == "__main__":
    main()
