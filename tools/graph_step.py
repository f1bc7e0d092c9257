"""Eager vs CUDA-graph replay of the bench step (per-layer evaluate pipeline)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dev = torch.device("cuda")
layers = bench.make_layers(dev, L, bench.TOKENS, 0)
for _ in range(3):
    bench.step(layers)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    bench.step(layers)
b.record()
torch.cuda.synchronize()
eager = a.elapsed_time(b) / 3 / L
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    bench.step(layers)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    outs = bench.step(layers)
g.replay()
torch.cuda.synchronize()
a.record()
for _ in range(3):
    g.replay()
b.record()
torch.cuda.synchronize()
graph = a.elapsed_time(b) / 3 / L
print(f"per layer: eager {eager:.3f} ms, graph {graph:.3f} ms")
