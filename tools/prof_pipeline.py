"""Profiling driver: the bench's per-layer pipeline (evaluate with ids_m=6 on
the oracle-gate workload, 1M tokens, DSV2L shape) run 3 times. Used plain and
under ncu (launch lists: -k regex:'moep|fix|dec_|predict|counters|split')."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
kind = sys.argv[2] if len(sys.argv) > 2 else "gate"
model, x, truth = W.make_layer(kind, 2048, 2048, 64, 6, n, seed=0, device="cuda")
dp = pb.DevicePredictor(model)
st = dp.new_status()
for _ in range(3):
    cnt, fc, ids = dp.evaluate(x, truth, 6, [6, 10, 64], ids_m=6, status=st)
torch.cuda.synchronize()
dp.check_status(st, x)
print("flagged", int(fc.item()))
