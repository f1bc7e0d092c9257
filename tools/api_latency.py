"""Cost of the numpy API path the reference binds: a
4,096-token predict_topk_batch at the DSV2L shape through the patched real
reference (baseline/_ref), split into the unavoidable x H2D (67 MB of fp64
from pageable numpy memory) and the device work (CUDA events around the same
call on a device-resident fp64 tensor: K0 cast + exactness check, K1, fix-up).
The model's weights stay resident across calls (predictor.device_for)."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import paper_2511_10676_b200 as pb  # noqa: E402
from paper_2511_10676_b200.integration import patch_reference  # noqa: E402
from paper_2511_10676_b200.predictor import device_for  # noqa: E402


def bf(a):
    m, e = np.frexp(np.asarray(a, dtype=np.float64))
    return np.ldexp(np.rint(m * 256.0), e - 8)


def main():
    import moepredict.predictor as P
    patch_reference()
    m = P.init_model("arch2", 2048, 2048, 64, seed=0)
    m.w1, m.w2 = bf(m.w1), bf(m.w2)
    x = bf(np.random.default_rng(0).standard_normal((4096, 2048)))
    for _ in range(3):
        P.predict_topk_batch(m, x, 6)
    torch.cuda.synchronize()
    walls = []
    for _ in range(20):
        t0 = time.perf_counter()
        P.predict_topk_batch(m, x, 6)
        walls.append((time.perf_counter() - t0) * 1e3)
    h2d = []
    for _ in range(20):
        t0 = time.perf_counter()
        xt = torch.from_numpy(x).cuda()
        torch.cuda.synchronize()
        h2d.append((time.perf_counter() - t0) * 1e3)
    dev = device_for(m)
    dev_ms = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dev.topk(xt, 6)
        b.record()
        torch.cuda.synchronize()
        dev_ms.append(a.elapsed_time(b))
    spec_ms = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dev.topk_speculative(xt, 6)
        b.record()
        torch.cuda.synchronize()
        spec_ms.append(a.elapsed_time(b))
    xb = xt.to(torch.bfloat16)
    bf_ms = []
    st = dev.new_status()
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dev.topk(xb, 6, status=st)
        b.record()
        torch.cuda.synchronize()
        bf_ms.append(a.elapsed_time(b))
    print(json.dumps({
        "call": "moepredict.predictor.predict_topk_batch(model, x[4096, 2048] fp64 numpy, 6), patched",
        "wall_ms_median": statistics.median(walls), "x_h2d_ms_median": statistics.median(h2d),
        "device_ms_fp64_input_median": statistics.median(dev_ms),
        "device_ms_numpy_path_median": statistics.median(spec_ms),
        "device_ms_bf16_resident_median": statistics.median(bf_ms),
        "weights_reuploaded_per_call": False}))


if __name__ == "__main__":
    main()
