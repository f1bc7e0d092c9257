"""Max K1 logit error / row scale for every K1 kernel on the shapes the margin
guard tests use (tests/test_gpu_parity.py::test_margin_covers_error*), against
torch float64 logits of the same bf16 inputs (a measurement tool)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_10676_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402


def ratio(model, x, lg):
    w1, w2 = (torch.as_tensor(t, device=x.device) for t in (model.w1, model.w2))
    b1, b2 = (torch.as_tensor(t, device=x.device) for t in (model.b1, model.b2))
    a = x.double() @ w1.T + b1
    h = a * torch.sigmoid(a)
    z = h @ w2.T + b2
    scale = torch.linalg.vector_norm(h, dim=1) * torch.linalg.vector_norm(w2, dim=1).max()
    return float(((lg.double() - z).abs().amax(1) / scale).max())


def main():
    dev = torch.device("cuda")
    cases = [(16384, 64, 2), (40000, 64, 4), (65536, 128, 4), (40000, 16, 4), (4096, 32, 1), (40000, 64, 5),
             (1 << 20, 64, 4), (1 << 20, 128, 4)]
    for n, e, kern in cases:
        d = h = 2048 if kern != 1 else 512
        if kern == 1:
            h = 384
        for kind in ("random", "gate"):
            if kind == "gate" and kern == 1:
                continue
            model, x, _ = W.make_layer(kind, d, h, e, 6 if e == 64 else 8, n, seed=5, device=dev)
            dp = pb.DevicePredictor(model, dev)
            lg = torch.empty((n, e), dtype=torch.float32, device=dev)
            dp._k1(x, logits=lg, kernel=kern)
            print(json.dumps({"n": n, "E": e, "kernel": kern, "kind": kind, "err_ratio_max": ratio(model, x, lg),
                              "kernel_tau_factor": 1.5 if (kern == 4 and e > 64) or kern == 1 else 1.0}), flush=True)
    # hidden split (small N)
    for n, e in ((256, 64), (4096, 64), (8192, 128), (300, 16)):
        model, x, _ = W.make_layer("random", 2048, 2048, e, 6, n, seed=6, device=dev)
        dp = pb.DevicePredictor(model, dev)
        lg = torch.empty((n, e), dtype=torch.float32, device=dev)
        dp._k1(x, logits=lg)
        print(json.dumps({"n": n, "E": e, "kernel": "split", "kind": "random", "err_ratio_max": ratio(model, x, lg)}),
              flush=True)


if __name__ == "__main__":
    main()
