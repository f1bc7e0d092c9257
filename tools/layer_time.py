"""Per-layer time of the bench pipeline (DevicePredictor.evaluate with ids_m = 6
on one oracle-gate DSV2L layer of 1 M tokens), CUDA events, median of 10; for
A/B of library builds: MOEP_LIB=<variant .so> python tools/layer_time.py"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

model, x, truth = W.make_layer("gate", 2048, 2048, 64, 6, 1 << 20, seed=0, device="cuda")
dp = pb.DevicePredictor(model)
st = dp.new_status()
for _ in range(3):
    cnt, fc, ids = dp.evaluate(x, truth, 6, [6, 10, 64], ids_m=6, status=st)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    cnt, fc, ids = dp.evaluate(x, truth, 6, [6, 10, 64], ids_m=6, status=st)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({"lib": os.environ.get("MOEP_LIB", "product"), "ms_median": statistics.median(ts), "ms_min": min(ts),
                  "flagged": int(fc.item()), "counters_sum": int(cnt.sum().item())}))
