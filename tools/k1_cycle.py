"""K1 alone: same layer repeated vs cycling over 8 layers (different x / weights)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

L = 8
dev = torch.device("cuda")
layers = bench.make_layers(dev, L, bench.TOKENS, 0)
ncnt = 2 + 2 * 3 + 2 * bench.E


def run(seq):
    part = torch.empty((148, ncnt), dtype=torch.int32, device=dev)
    for li in seq[:2]:
        _, dp, x, t = layers[li]
        dp._k1(x, m_sel=0, bounds=(1, 6, 10), truth=t, k=6, m_values=bench.M_LIST, partials=part)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for li in seq:
        _, dp, x, t = layers[li]
        dp._k1(x, m_sel=0, bounds=(1, 6, 10), truth=t, k=6, m_values=bench.M_LIST, partials=part)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / len(seq)


print("same layer x16:", round(run([0] * 16), 3), "ms")
print("cycle 8 layers x2:", round(run(list(range(8)) * 2), 3), "ms")
print("same layer x16 again:", round(run([3] * 16), 3), "ms")
