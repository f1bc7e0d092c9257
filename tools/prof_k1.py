"""Profiling driver: K1 (+K2 fix-up) on one DSV2L layer, 1M tokens. Used plain and under ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
layers = bench.make_layers(torch.device("cuda"), 1, n, 0)
model, dp, x, truth = layers[0]
for _ in range(3):
    cnt, fc, _ = dp.evaluate(x, truth, 6, [6, 10, 64], ids_m=6)
torch.cuda.synchronize()
print("flagged", int(fc.item()), "k1 ms", bench.time_k1(dp, x, truth, reps=3))
