"""Where the per-layer evaluate time goes inside the bench step (CUDA events
between the pipeline stages, steady state, 8 layers)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2511_10676_b200 import engine  # noqa: E402

L = 8
dev = torch.device("cuda")
layers = bench.make_layers(dev, L, bench.TOKENS, 0)
marks = []
orig_k1, orig_fix = engine.DevicePredictor._k1, engine.DevicePredictor._fixup


def ev(tag):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks.append((tag, e))


def k1(self, *a, **kw):
    ev("start")
    r = orig_k1(self, *a, **kw)
    ev("k1")
    return r


def fix(self, *a, **kw):
    r = orig_fix(self, *a, **kw)
    ev("fixup")
    return r


engine.DevicePredictor._k1, engine.DevicePredictor._fixup = k1, fix
for _ in range(3):
    bench.step(layers)
torch.cuda.synchronize()
marks.clear()
for _ in range(2):
    bench.step(layers)
ev("end")
torch.cuda.synchronize()
acc = {}
for (t0, e0), (t1, e1) in zip(marks, marks[1:]):
    key = f"{t0}->{t1}"
    acc.setdefault(key, []).append(e0.elapsed_time(e1))
for k, v in acc.items():
    print(f"{k:20s} n={len(v):3d} mean={sum(v) / len(v):.3f} ms")
