"""One K1 v4 launch then one K1 v5 launch on the same 1M-token DSV2L layer
(ncu driver: ncu -k regex:"predict_(pair|quad)" -c 2 python tools/prof_k1v5.py)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_10676_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402


def main():
    dev = torch.device("cuda")
    model, x, truth = W.make_layer("gate", 2048, 2048, 64, 6, 1 << 20, seed=1, device=dev)
    dp = pb.DevicePredictor(model, dev)
    part = torch.empty((dp.n_sms, 2 + 6 + 128), dtype=torch.int32, device=dev)
    ids = torch.empty((x.shape[0], 6), dtype=torch.int32, device=dev)
    for kv in (4, 5):
        dp.k1_kernel = kv
        dp._k1(x, m_sel=6, bounds=(1, 6, 10), ids=ids, truth=truth, k=6, m_values=[6, 10, 64], partials=part)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
