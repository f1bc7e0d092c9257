"""Launch list of one decode-batch predictor call (for ncu): Qwen3 shape."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
from oracle import oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
force_k1 = len(sys.argv) > 2 and sys.argv[2] == "k1"
E = int(sys.argv[3]) if len(sys.argv) > 3 else 128
m = pb.init_model("arch2", 2048, 2048, E, seed=1)
m.w1, m.w2 = O.round_bf16(m.w1), O.round_bf16(m.w2)
dev = m.to_device()
if force_k1:
    dev.decode_max_tokens = 0
x = torch.randn((n, 2048), device="cuda").to(torch.bfloat16)
for _ in range(3):
    dev.topk(x, 8 if E == 128 else 6, validate=False)
torch.cuda.synchronize()
print("ok")
