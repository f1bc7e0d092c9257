"""Generate golden fixtures by running the REAL reference (`moepredict`) in the
build container. The reference lives at /root/reference and does not exist on
the GPU box, so its outputs are frozen here as small .npz files that
tests/test_oracle_golden.py (CPU) and the -m gpu parity tests consume.

Run:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [synthgen]
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from moepredict import core, losses, metrics, predictor  # noqa: E402
from moepredict.trainer import TrainConfig, _Optimizer  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from trace_corrupt import corruptions as _corruptions  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def bf16_round(x):
    # same rule as oracle.round_bf16, repeated here so this script only depends on the reference
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    return np.ldexp(np.rint(m * 256.0), e - 8)


def topk_cases():
    rng = np.random.default_rng(1)
    out = {}
    # forced ties, signed zeros, wide magnitudes
    s = rng.choice([0.0, -0.0, 0.25, 0.5, 1.0, -1.0], size=(300, 11))
    out["tie_scores"] = s
    for k in (1, 3, 6, 11):
        out[f"tie_top{k}"] = core.top_k_batch(s, k)
    s2 = rng.standard_normal((300, 64))
    out["rand_scores"] = s2
    for k in (1, 6, 10, 64):
        out[f"rand_top{k}"] = core.top_k_batch(s2, k)
    out["rand_order"] = core.rank_order(s2)
    return out


def predictor_cases():
    rng = np.random.default_rng(2)
    out = {}
    # reference-test shape: d=8, h=16, E=8 perturbed models (test_predictor.py:21-28)
    for arch in ("arch1", "arch2"):
        model = predictor.init_model(arch, 8, 16, 8, seed=7)
        for p in model.param_dict().values():
            p += 0.3 * rng.standard_normal(p.shape)
        if arch == "arch1":
            model.bn_mean += 0.1 * rng.standard_normal(16)
            model.bn_var = np.abs(model.bn_var + 0.2 * rng.standard_normal(16))
        x = rng.standard_normal((32, 8))
        pre = f"small_{arch}_"
        for name in ("w1", "b1", "w2", "b2"):
            out[pre + name] = getattr(model, name)
        if arch == "arch1":
            for name in ("bn_scale", "bn_shift", "bn_mean", "bn_var"):
                out[pre + name] = getattr(model, name)
        out[pre + "x"] = x
        out[pre + "logits"] = predictor.predict_logits(model, x)
        out[pre + "top3"] = predictor.predict_topk_batch(model, x, 3)
        dz = rng.standard_normal((32, 8))
        g = predictor.backward(model, x, dz)
        out[pre + "dz"] = dz
        for name, v in g.items():
            out[pre + "grad_" + name] = v
    # bf16-representable C1-shaped layer (init_model seed 0, weights rounded to bf16)
    model = predictor.init_model("arch2", 2048, 2048, 64, seed=0)
    model.w1 = bf16_round(model.w1)
    model.w2 = bf16_round(model.w2)
    x = bf16_round(rng.standard_normal((256, 2048)))
    out["c1_x"] = x.astype(np.float32)  # exact: bf16 values
    out["c1_logits"] = predictor.predict_logits(model, x)
    out["c1_top6"] = predictor.predict_topk_batch(model, x, 6)
    out["c1_top10"] = predictor.predict_topk_batch(model, x, 10)
    # init stream check: a slice of the reference init (seed 0 and 3)
    m0 = predictor.init_model("arch2", 2048, 2048, 64, seed=0)
    out["init_s0_w1_head"] = m0.w1[:4, :16].copy()
    out["init_s0_w2_tail"] = m0.w2[-2:, -16:].copy()
    m3 = predictor.init_model("arch1", 12, 30, 7, seed=3)
    out["init_s3_w1"] = m3.w1
    out["init_s3_w2"] = m3.w2
    return out


def loss_cases():
    rng = np.random.default_rng(3)
    out = {}
    for n, e, k in ((4, 8, 2), (16, 16, 2), (8, 64, 6)):
        scores = core.softmax(rng.standard_normal((n, e)), axis=1)
        labels = losses.BatchLabels.from_scores(scores, k)
        z = rng.standard_normal((n, e))
        pre = f"n{n}e{e}k{k}_"
        out[pre + "scores"] = scores
        out[pre + "z"] = z
        out[pre + "rank_of"] = labels.rank_of
        out[pre + "mask"] = labels.topk_mask
        for fam in ("mse", "wbce", "focal", "ranking"):
            loss, grad = losses.loss_and_grad(losses.LossSpec(family=fam), z, labels)
            out[pre + fam + "_loss"] = np.float64(loss)
            out[pre + fam + "_grad"] = grad
        _, _, n_pairs = losses.ranking_hinge(z, labels)
        out[pre + "n_pairs"] = np.int64(n_pairs)
    return out


def metric_cases():
    rng = np.random.default_rng(4)
    out = {}
    for idx, (n, e, k) in enumerate(((200, 12, 3), (500, 64, 6), (300, 128, 8), (100, 16, 2))):
        z = rng.standard_normal((n, e))
        z[::7, 1] = z[::7, 0]  # ties
        truth = np.sort(rng.permuted(np.tile(np.arange(e), (n, 1)), axis=1)[:, :k], axis=1)
        ms = metrics.default_m_list(k, e)
        res = metrics.evaluate_predictions(z, truth, e)
        pre = f"m{idx}_"
        out[pre + "z"] = z
        out[pre + "truth"] = truth
        out[pre + "m_list"] = np.array(ms)
        out[pre + "exact"] = np.float64(res.exact_match)
        out[pre + "top1"] = np.float64(res.top1)
        out[pre + "overprov"] = np.array([res.overprov[m] for m in ms])
        out[pre + "recall"] = np.array([res.overprov_recall[m] for m in ms])
        out[pre + "hits"] = res.per_expert_hits
        out[pre + "truthc"] = res.per_expert_truth
    return out


def adam_cases():
    rng = np.random.default_rng(5)
    out = {}
    params = {"w": rng.standard_normal((6, 5)), "b": rng.standard_normal(5)}
    out["p0_w"], out["p0_b"] = params["w"].copy(), params["b"].copy()
    for opt, lr in (("adam", 1e-3), ("sgd", 0.05), ("momentum", 0.02)):
        p = {n: v.copy() for n, v in params.items()}
        o = _Optimizer(TrainConfig(optimizer=opt, learning_rate=lr), p)
        for t in range(3):
            g = {"w": rng.standard_normal((6, 5)), "b": rng.standard_normal(5)}
            out[f"{opt}_g{t}_w"], out[f"{opt}_g{t}_b"] = g["w"], g["b"]
            o.step(p, g)
        out[f"{opt}_p3_w"], out[f"{opt}_p3_b"] = p["w"], p["b"]
    return out


def trace_cases():
    """MOEPA1 files written / read by the reference (synthgen.py:197-253)."""
    import tempfile
    from moepredict import synthgen, exceptions
    rng = np.random.default_rng(7)
    d, e, k = 32, 16, 4
    router = core.RouterSpec(d, e, k, rng.standard_normal((e, d)) / np.sqrt(d))
    teacher = synthgen.TeacherSpec(router, transform="nonlinear", noise_sigma=0.1, seed=5)
    data = synthgen.generate_dataset(teacher, 200)
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "t.moepa")
        synthgen.write_trace(path, data)
        blob = open(path, "rb").read()
        with open(os.path.join(HERE, "trace_small.moepa"), "wb") as f:
            f.write(blob)
        back = synthgen.read_trace(path)
        out["acts"], out["scores"], out["topk"] = back.activations, back.true_scores, back.true_topk
        out["dims"] = np.array([d, e, k, len(back)])
        # ties: scores with exact equal values (lower index must win)
        sc = np.zeros((64, 8), dtype=np.float64)
        sc[:, :4] = 0.25
        sc[32:] = rng.dirichlet(np.ones(8), size=32)
        sc[40:48, 2] = sc[40:48, 5]
        sc = sc / sc.sum(axis=1, keepdims=True)
        tie = synthgen.make_dataset(rng.standard_normal((64, 8)), sc, 3)
        synthgen.write_trace(path, tie)
        with open(os.path.join(HERE, "trace_ties.moepa"), "wb") as f:
            f.write(open(path, "rb").read())
        out["tie_topk"] = synthgen.read_trace(path).true_topk
        # corruptions: the exception class the reference raises for each
        names, kinds, msgs = [], [], []
        for name, bad in _corruptions(blob, d, e, k).items():
            with open(path, "wb") as f:
                f.write(bad)
            try:
                synthgen.read_trace(path)
                kind = "ok"
            except exceptions.MoePredictError as exc:
                kind = type(exc).__name__
                msgs.append(str(exc))
            else:
                msgs.append("")
            names.append(name)
            kinds.append(kind)
        out["corrupt_names"] = np.array(names)
        out["corrupt_kinds"] = np.array(kinds)
        out["corrupt_msgs"] = np.array(msgs)
    return out


SYNTH_CASES = [
    # name, d, E, k, n, seed, transform, post_norm, noise_sigma, nonlinear_hidden
    ("dsv2l_identity", 2048, 64, 6, 24, 3, "identity", True, 0.0, 64),
    ("nonlinear_noise", 256, 16, 2, 40, 5, "nonlinear", True, 0.1, 32),
    ("linear_raw", 128, 128, 8, 24, 7, "linear", False, 0.0, 64),
    ("identity_noise_raw", 96, 8, 3, 30, 11, "identity", False, 0.25, 64),
]


def synthgen_cases():
    """synthgen.generate_dataset (synthgen.py:162-189) of the real reference
    for four teachers (transforms, noise, post_norm on/off, odd d)."""
    from moepredict import synthgen
    out = {}
    for name, d, e, k, n, seed, transform, post_norm, sigma, nh in SYNTH_CASES:
        gate = np.random.default_rng(seed + 100).standard_normal((e, d)) / np.sqrt(d)
        router = core.RouterSpec(d, e, k, gate)
        teacher = synthgen.TeacherSpec(router, transform=transform, post_norm=post_norm, noise_sigma=sigma,
                                       nonlinear_hidden=nh, seed=seed)
        data = synthgen.generate_dataset(teacher, n)
        out[name + "_gate"] = gate
        out[name + "_x"] = data.activations
        out[name + "_scores"] = data.true_scores
        out[name + "_topk"] = data.true_topk
        # raw fp64 normals of the first 2 samples (activation then noise row)
        raw = []
        for i in range(2):
            g = synthgen._rng(seed, i)
            raw.append(g.standard_normal(2 * d))
        out[name + "_raw"] = np.stack(raw)
    # layer_norm of wide-magnitude rows (numpy reduction order)
    rng = np.random.default_rng(9)
    for d in (2048, 1000, 129, 7):
        x = rng.standard_normal((6, d)) * np.exp(2 * rng.standard_normal((6, d))) + 3.0
        out[f"ln_{d}_x"] = x
        out[f"ln_{d}_y"] = core.layer_norm(x)
    return out


def main():
    if sys.argv[1:] == ["synthgen"]:
        np.savez_compressed(os.path.join(HERE, "synthgen.npz"), **synthgen_cases())
        print("synthgen.npz", os.path.getsize(os.path.join(HERE, "synthgen.npz")))
        return
    np.savez_compressed(os.path.join(HERE, "topk.npz"), **topk_cases())
    np.savez_compressed(os.path.join(HERE, "predictor.npz"), **predictor_cases())
    np.savez_compressed(os.path.join(HERE, "losses.npz"), **loss_cases())
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **metric_cases())
    np.savez_compressed(os.path.join(HERE, "optim.npz"), **adam_cases())
    np.savez_compressed(os.path.join(HERE, "trace.npz"), **trace_cases())
    np.savez_compressed(os.path.join(HERE, "synthgen.npz"), **synthgen_cases())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
