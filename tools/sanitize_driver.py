"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck,
one tool per run): every kernel family of the hot path once, checked against
the oracle so a silent corruption would also fail here.

  K0 norm (fast + general) | K1 v4 / v2 (split) / 1-SM + K2 fix-up (GEMM and
  split-hidden) + counters reduce | decode fp64 | K7 eval / top-k / ranks |
  K3 labels, K4 loss, K5, K6 (one fp32 + one fp64 training step) |
  K8 plan + K9 gather + commit | K10 trace ingest | K11 teacher | DGEMM

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker)


def main():
    rng = np.random.default_rng(0)
    dev = "cuda"
    # K0
    from paper_2511_10676_b200.engine import input_norm, eval_logits_device, rank_order_device
    for d in (512, 1000):
        x = O.round_bf16(rng.standard_normal((97, d)))
        g = rng.uniform(0.5, 1.5, d)
        out = input_norm(torch.from_numpy(x).to(dev, torch.bfloat16), "rmsnorm", g)
        assert np.array_equal(out.double().cpu().numpy(), O.input_norm_bf16(x, "rmsnorm", g))
    # K1 (three kernels) + K2 + counters
    for (d, h, e, n, kern) in ((256, 512, 64, 40000, 4), (256, 512, 64, 700, 2), (256, 384, 32, 900, 1)):
        m = pb.init_model("arch2", d, h, e, seed=1)
        m.w1, m.w2 = O.round_bf16(m.w1), O.round_bf16(m.w2)
        x = O.round_bf16(rng.standard_normal((n, d)))
        zr = O.predict_logits({"arch": "arch2", "w1": m.w1, "b1": m.b1, "w2": m.w2, "b2": m.b2}, x)
        dp = pb.DevicePredictor(m, dev, tau_rel=2e-4)  # wide margin: the fix-up kernels all run
        dp.decode_max_tokens = 0
        xt = torch.from_numpy(x).to(dev, torch.bfloat16)
        truth = O.top_k_batch(zr + 0.05 * rng.standard_normal(zr.shape), 6)
        cnt, fc, ids = dp.evaluate(xt, torch.from_numpy(truth), 6, [6, 10, e], ids_m=6)
        assert np.array_equal(ids.cpu().numpy(), O.top_k_batch(zr, 6)), (d, h, e, n)
        c = pb.EvalCounters.from_array(cnt.cpu().numpy(), 6, e, [6, 10, e])
        assert c.overprov == O.eval_counters(zr, truth, e, [6, 10, e])["overprov_count"]
        z = eval_logits_device(torch.from_numpy(zr).to(dev), torch.from_numpy(truth), 6, e, [6, 10])
        rank_order_device(torch.from_numpy(zr).to(dev))
        dp.topk(xt[:5], 6)  # decode kernel
        torch.cuda.synchronize()
    # training: fp32 and fp64 steps
    for prec in ("fp32", "fp64"):
        m = pb.init_model("arch2", 256, 256, 16, seed=2)
        m.w1, m.w2 = O.round_bf16(m.w1), O.round_bf16(m.w2)
        tr = pb.DeviceTrainer(m, pb.LossSpec("ranking"), precision=prec)
        x = torch.from_numpy(O.round_bf16(rng.standard_normal((512, 256)))).to(dev)
        s = torch.softmax(torch.randn(512, 16, device=dev, dtype=torch.float64), 1)
        lab = pb.BatchLabels.from_scores(s, 2)
        sd = torch.float64 if prec == "fp64" else torch.float32
        tr.step(x if prec == "fp64" else x.to(torch.bfloat16), lab.true_scores.to(sd), lab.topk_mask.to(torch.uint8),
                lab.rank_of)
        torch.cuda.synchronize()
    # prefetch
    from paper_2511_10676_b200 import prefetch as pf
    store, cache = pf.ExpertStore(16, 1 << 16), pf.ExpertCache(8, 1 << 16, 16)
    p = pf.Prefetcher(store, cache)
    p.load_sm_gather(torch.tensor([[1, 5], [5, 9]], dtype=torch.int32, device=dev), 8)
    p.load_copy_engine(torch.tensor([[2, 9]], dtype=torch.int32, device=dev))
    torch.cuda.synchronize()
    # trace ingest + teacher + dgemm
    from paper_2511_10676_b200 import synthgen as sg, trace_io
    t = sg.TeacherSpec(sg.RouterSpec(64, 8, 2, rng.standard_normal((8, 64)) / 8.0), transform="nonlinear",
                       nonlinear_hidden=32, seed=1)
    data = sg.generate_dataset(t, 300)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "t.moepa")
        trace_io.write_trace(path, data)
        back = trace_io.read_trace_device(path)
        assert np.array_equal(back.to_host().true_topk, data.true_topk)
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
