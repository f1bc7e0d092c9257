"""Ad-hoc GPU bring-up check (not part of the test suite): K1/K2/K7 vs the oracle."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10676_b200 as pb  # noqa: E402
from oracle import oracle as O  # noqa: E402

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def small():
    g = np.load(os.path.join(G, "predictor.npz"))
    for arch in ("arch1", "arch2"):
        pre = f"small_{arch}_"
        kw = {}
        if arch == "arch1":
            kw = {n: g[pre + n] for n in ("bn_scale", "bn_shift", "bn_mean", "bn_var")}
        m = pb.PredictorModel(arch, g[pre + "w1"], g[pre + "b1"], g[pre + "w2"], g[pre + "b2"], **kw)
        z = pb.predict_logits(m, g[pre + "x"])
        ids = pb.predict_topk_batch(m, g[pre + "x"], 3)
        print(arch, "small logits maxerr", np.abs(z - g[pre + "logits"]).max(),
              "ids equal", np.array_equal(ids, g[pre + "top3"]))


def c1():
    g = np.load(os.path.join(G, "predictor.npz"))
    m = pb.init_model("arch2", 2048, 2048, 64, seed=0)
    m.w1 = O.round_bf16(m.w1)
    m.w2 = O.round_bf16(m.w2)
    x = g["c1_x"].astype(np.float64)
    dev = m.to_device()
    xt = torch.from_numpy(x).cuda()
    z, flags = dev.logits(xt, return_flags=True)
    z = z.cpu().numpy()
    print("c1 golden logits maxerr", np.abs(z - g["c1_logits"]).max(), "flagged", int(flags.sum()))
    for mm, key in ((6, "c1_top6"), (10, "c1_top10")):
        ids = dev.topk(xt, mm).cpu().numpy()
        print(f"c1 top{mm} equal", np.array_equal(ids, g[key]))


def big(n=32768, e=64, k=6, arch="arch2", d=2048, h=2048, seed=1):
    rng = np.random.default_rng(seed)
    m = pb.init_model(arch, d, h, e, seed=seed)
    m.w1 = O.round_bf16(m.w1)
    m.w2 = O.round_bf16(m.w2)
    if arch == "arch1":
        m.bn_mean = rng.standard_normal(h) * 0.05
        m.bn_var = 0.3 + rng.random(h) * 0.5
        m.bn_scale = 1 + 0.1 * rng.standard_normal(h)
        m.bn_shift = 0.1 * rng.standard_normal(h)
    x = O.round_bf16(rng.standard_normal((n, d)))
    p = {"arch": arch, "w1": m.w1, "b1": m.b1, "w2": m.w2, "b2": m.b2}
    if arch == "arch1":
        p.update(bn_scale=m.bn_scale, bn_shift=m.bn_shift, bn_mean=m.bn_mean, bn_var=m.bn_var)
    t0 = time.time()
    zref, cache = O.forward_eval(p, x)
    tcpu = time.time() - t0
    dev = m.to_device()
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    # raw K1 logits (pre fix-up) for the error model
    xb = xt
    lg = torch.empty((n, e), dtype=torch.float32, device="cuda")
    flags, fl, fc = dev._k1(xb, logits=lg, m_sel=k, bounds=(1, k, k + 4),
                            ids=torch.empty((n, k), dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    z1 = lg.double().cpu().numpy()
    err = np.abs(z1 - zref)
    hn = np.linalg.norm(cache["h"], axis=1)
    scale = hn * np.linalg.norm(m.w2, axis=1).max()
    rel = err.max(axis=1) / scale
    print(f"{arch} E={e} n={n}: K1 raw maxerr {err.max():.3e}, max err/scale {rel.max():.3e}, "
          f"flagged {int(fc.item())} ({fc.item()/n:.2e}), cpu oracle {tcpu:.1f}s")
    ids = dev.topk(xt, k).cpu().numpy()
    ref_ids = O.top_k_batch(zref, k)
    print("  ids equal", np.array_equal(ids, ref_ids), "mismatching rows", int((ids != ref_ids).any(axis=1).sum()))
    truth = np.sort(rng.permuted(np.tile(np.arange(e), (n, 1)), axis=1)[:, :k], axis=1)
    # make truth correlated with predictions so counters are non-trivial
    truth[: n // 2] = ref_ids[: n // 2]
    ms = O.default_m_list(k, e)
    cnt, fcount, _ = dev.evaluate(xt, torch.from_numpy(truth), k, ms)
    c = pb.EvalCounters.from_array(cnt.cpu().numpy(), k, e, sorted(set(ms) | {k}))
    oc = O.eval_counters(zref, truth, e, ms)
    ok = (c.n == oc["n"] and c.top1 == oc["top1_count"] and c.overprov == oc["overprov_count"]
          and c.recall == oc["recall_count"] and np.array_equal(c.per_expert_hits, oc["per_expert_hits"])
          and np.array_equal(c.per_expert_truth, oc["per_expert_truth"]))
    print("  counters equal", ok, "flagged(eval)", int(fcount.item()))
    if not ok:
        print("   gpu", c.n, c.top1, c.overprov, c.recall)
        print("   ref", oc["n"], oc["top1_count"], oc["overprov_count"], oc["recall_count"])


def timing(n=1 << 20, e=64, d=2048, h=2048):
    m = pb.init_model("arch2", d, h, e, seed=0)
    m.w1 = O.round_bf16(m.w1)
    m.w2 = O.round_bf16(m.w2)
    dev = m.to_device()
    xb = torch.randn((n, d), device="cuda").to(torch.bfloat16)
    ids = torch.empty((n, 6), dtype=torch.int32, device="cuda")
    for _ in range(3):
        dev._k1(xb, m_sel=6, bounds=(1, 6, 10), ids=ids)
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    reps = 5
    for _ in range(reps):
        dev._k1(xb, m_sel=6, bounds=(1, 6, 10), ids=ids)
    t.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(t) / reps
    flops = 2 * n * (d * h + h * e)
    print(f"K1 n={n}: {ms:.3f} ms  {n/ms/1e3:.1f} M tok/s  {flops/ms/1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    what = sys.argv[1:] or ["small", "c1", "big", "timing"]
    for w in what:
        if w == "big":
            big()
            big(n=16384, e=128, k=8)
            big(n=16384, e=16, k=2, d=4096)
            big(n=8192, e=64, k=6, arch="arch1")
        else:
            globals()[w]()
