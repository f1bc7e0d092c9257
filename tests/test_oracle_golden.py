"""Pin the CPU oracle (oracle/oracle.py) before trusting it as the checker.

(a) known-answer values from the reference's own tests (file:line cited);
(b) golden fixtures produced by running the real reference
    (tests/golden/make_golden.py).
"""

import os

import numpy as np
import pytest

from conftest import central_diff, rel_error
from oracle import oracle as O


# ----------------------------------------------------------- known answers
class TestKnownAnswers:
    def test_top_k_hand_cases(self):
        # test_core.py:60-64, 78-79
        assert O.top_k(np.array([0.1, 0.7, 0.2]), 1).tolist() == [1]
        assert O.top_k(np.array([0.5, 0.5, 0.0]), 1).tolist() == [0]
        assert O.top_k(np.array([0.4, 0.1, 0.3, 0.2]), 2).tolist() == [0, 2]

    def test_top_k_sort_oracle(self, rng):
        # test_core.py:66-76: stable sort by (-score, index), forced ties
        for _ in range(200):
            n = int(rng.integers(2, 12))
            k = int(rng.integers(1, n + 1))
            s = rng.choice([0.0, 0.25, 0.5, 1.0], size=n)
            want = sorted(sorted(range(n), key=lambda i: (-s[i], i))[:k])
            assert O.top_k(s, k).tolist() == want

    def test_signed_zero_ties(self):
        # -0.0 and +0.0 tie -> lower index wins (SURVEY §0 finding 3)
        assert O.top_k(np.array([-0.0, 0.0, -1.0]), 1).tolist() == [0]
        assert O.top_k(np.array([0.0, -0.0, -1.0]), 1).tolist() == [0]

    def test_silu_hand_value(self):
        # test_predictor.py:38-48: SiLU(2) = 2 sigma(2) = 1.7616
        assert O.silu(np.array([2.0]))[0] == pytest.approx(1.7616, abs=1e-4)

    def test_activation_formulas(self):
        u = np.linspace(-4, 4, 101)
        assert np.allclose(O.silu(u), u / (1 + np.exp(-u)), atol=1e-12)
        ref = 0.5 * u * (1 + np.tanh(np.sqrt(2 / np.pi) * (u + 0.044715 * u**3)))
        assert np.allclose(O.gelu_tanh(u), ref, atol=1e-6)

    def test_wbce_hand_value(self):
        # test_losses.py:78-83: E=2, k=1, zero logits -> 3 ln 2
        lab = O.batch_labels(np.array([[0.9, 0.1]]), 1)
        loss, _ = O.loss_and_grad({"family": "wbce"}, np.zeros((1, 2)), lab)
        assert loss == pytest.approx(3.0 * np.log(2.0), abs=1e-12)

    def test_hinge_equal_logits(self):
        # test_losses.py:133-137
        lab = O.batch_labels(np.array([[0.7, 0.3]]), 1)
        h, _, n_pairs = O.ranking_hinge(np.ones((1, 2)), lab, margin=0.1)
        assert n_pairs == 1 and h == pytest.approx(0.1)

    def test_hinge_tie_exclusion(self):
        # test_losses.py:159-168
        lab = {"true_scores": np.array([[0.4, 0.4, 0.2]]),
               "topk_mask": np.array([[True, True, False]]), "rank_of": np.array([[1, 2, 3]])}
        _, _, n_pairs = O.ranking_hinge(np.zeros((1, 3)), lab)
        assert n_pairs == 2

    def test_recall_vs_coverage(self):
        # test_metrics.py:121-128
        res = O.evaluate_predictions(np.array([[3.0, 2.0, 1.0, 0.0]]), np.array([[0, 3]]), 4, [2, 4])
        assert res["overprov"][2] == 0.0 and res["overprov_recall"][2] == 0.5 and res["overprov"][4] == 1.0

    def test_per_expert_counts(self):
        # test_metrics.py:130-136
        z = np.array([[3.0, 2.0, 1.0, 0.0], [0.0, 1.0, 2.0, 3.0]])
        res = O.evaluate_predictions(z, np.array([[0, 1], [0, 3]]), 4)
        assert res["per_expert_truth"].tolist() == [2, 1, 0, 1]
        assert res["per_expert_hits"].tolist() == [1, 1, 0, 1]

    def test_param_count(self):
        # test_predictor.py:176-179 and SURVEY A1: 4,327,488 at the C1 shape
        p = O.init_params("arch2", 12, 30, 7)
        assert sum(p[n].size for n in ("w1", "b1", "w2", "b2")) == 30 * (12 + 7) + 30 + 7
        assert 2048 * (2048 + 64) + 2048 + 64 == 4_327_488

    def test_bf16_rounding(self):
        x = np.array([1.0, 1.0 + 2**-8, 1.0 + 3 * 2**-9, -2.5, 1e-40, 3.0e38 * 1.2])
        r = O.round_bf16(x)
        assert r[0] == 1.0
        assert r[1] == 1.0  # halfway -> even
        assert r[2] == 1.0 + 2**-7  # above halfway rounds up
        assert r[3] == -2.5
        assert np.isinf(r[5])
        # already-bf16 values are fixed points
        y = O.round_bf16(np.random.default_rng(0).standard_normal(1000))
        assert np.array_equal(O.round_bf16(y), y)


# ------------------------------------------------------- reference goldens
def test_topk_golden(golden):
    g = golden("topk")
    for k in (1, 3, 6, 11):
        assert np.array_equal(O.top_k_batch(g["tie_scores"], k), g[f"tie_top{k}"])
    for k in (1, 6, 10, 64):
        assert np.array_equal(O.top_k_batch(g["rand_scores"], k), g[f"rand_top{k}"])
    assert np.array_equal(O.rank_order(g["rand_scores"]), g["rand_order"])


@pytest.mark.parametrize("arch", ["arch1", "arch2"])
def test_predictor_golden(golden, arch):
    g = golden("predictor")
    pre = f"small_{arch}_"
    p = {"arch": arch, **{n: g[pre + n] for n in ("w1", "b1", "w2", "b2")}}
    if arch == "arch1":
        p.update({n: g[pre + n] for n in ("bn_scale", "bn_shift", "bn_mean", "bn_var")})
    z, cache = O.forward_eval(p, g[pre + "x"])
    assert np.allclose(z, g[pre + "logits"], rtol=0, atol=1e-12)
    assert np.array_equal(O.top_k_batch(z, 3), g[pre + "top3"])
    grads = O.backward_eval(p, cache, g[pre + "dz"])
    for name, v in grads.items():
        assert np.allclose(v, g[pre + "grad_" + name], rtol=1e-10, atol=1e-12), name


def test_c1_golden(golden):
    g = golden("predictor")
    p = O.init_params("arch2", 2048, 2048, 64, seed=0)
    p["w1"], p["w2"] = O.round_bf16(p["w1"]), O.round_bf16(p["w2"])
    z = O.predict_logits(p, g["c1_x"].astype(np.float64))
    assert np.allclose(z, g["c1_logits"], rtol=0, atol=1e-12)
    assert np.array_equal(O.top_k_batch(z, 6), g["c1_top6"])
    assert np.array_equal(O.top_k_batch(z, 10), g["c1_top10"])


def test_init_stream_matches_reference(golden):
    g = golden("predictor")
    p0 = O.init_params("arch2", 2048, 2048, 64, seed=0)
    assert np.array_equal(p0["w1"][:4, :16], g["init_s0_w1_head"])
    assert np.array_equal(p0["w2"][-2:, -16:], g["init_s0_w2_tail"])
    p3 = O.init_params("arch1", 12, 30, 7, seed=3)
    assert np.array_equal(p3["w1"], g["init_s3_w1"]) and np.array_equal(p3["w2"], g["init_s3_w2"])


def test_losses_golden(golden):
    g = golden("losses")
    for n, e, k in ((4, 8, 2), (16, 16, 2), (8, 64, 6)):
        pre = f"n{n}e{e}k{k}_"
        lab = O.batch_labels(g[pre + "scores"], k)
        assert np.array_equal(lab["rank_of"], g[pre + "rank_of"])
        assert np.array_equal(lab["topk_mask"], g[pre + "mask"])
        for fam in ("mse", "wbce", "focal", "ranking"):
            loss, grad = O.loss_and_grad({"family": fam}, g[pre + "z"], lab)
            assert loss == pytest.approx(float(g[pre + fam + "_loss"]), rel=1e-12, abs=1e-15), fam
            assert np.allclose(grad, g[pre + fam + "_grad"], rtol=1e-10, atol=1e-15), fam
        _, _, n_pairs = O.ranking_hinge(g[pre + "z"], lab)
        assert n_pairs == int(g[pre + "n_pairs"])


def test_metrics_golden(golden):
    g = golden("metrics")
    for idx in range(4):
        pre = f"m{idx}_"
        e = g[pre + "z"].shape[1]
        ms = g[pre + "m_list"].tolist()
        res = O.evaluate_predictions(g[pre + "z"], g[pre + "truth"], e, ms)
        assert res["exact_match"] == float(g[pre + "exact"])
        assert res["top1"] == float(g[pre + "top1"])
        assert [res["overprov"][m] for m in ms] == g[pre + "overprov"].tolist()
        assert [res["overprov_recall"][m] for m in ms] == g[pre + "recall"].tolist()
        assert np.array_equal(res["per_expert_hits"], g[pre + "hits"])
        assert np.array_equal(res["per_expert_truth"], g[pre + "truthc"])


def test_optim_golden(golden):
    g = golden("optim")
    for opt, lr in (("adam", 1e-3), ("sgd", 0.05), ("momentum", 0.02)):
        params = {"w": g["p0_w"].copy(), "b": g["p0_b"].copy()}
        state = {}
        for t in range(3):
            grads = {"w": g[f"{opt}_g{t}_w"], "b": g[f"{opt}_g{t}_b"]}
            if opt == "adam":
                O.adam_step(params, grads, state, t + 1, lr=lr)
            else:
                O.sgd_step(params, grads, state, lr, momentum=0.9 if opt == "momentum" else None)
        assert np.array_equal(params["w"], g[f"{opt}_p3_w"]), opt
        assert np.array_equal(params["b"], g[f"{opt}_p3_b"]), opt


def test_oracle_gradients_fd(rng):
    # analytic oracle gradients vs central differences (test_acceptance.py:37-97 style)
    for arch in ("arch1", "arch2"):
        p = O.init_params(arch, 8, 16, 8, seed=int(rng.integers(1 << 30)))
        for n in ("w1", "b1", "w2", "b2"):
            p[n] = p[n] + 0.3 * rng.standard_normal(p[n].shape)
        x = rng.standard_normal((4, 8))
        lab = O.batch_labels(O.softmax(rng.standard_normal((4, 8)), axis=1), 2)
        for fam in ("mse", "wbce", "focal"):
            spec = {"family": fam}
            z, cache = O.forward_eval(p, x)
            _, dz = O.loss_and_grad(spec, z, lab)
            grads = O.backward_eval(p, cache, dz)
            params = {n: p[n] for n in ("w1", "b1", "w2", "b2")}
            fd = central_diff(lambda: O.loss_and_grad(spec, O.predict_logits(p, x), lab)[0], params)
            for name in params:
                assert rel_error(grads[name], fd[name]) < 1e-4, (arch, fam, name)


# ------------------------------------------------------------ MOEPA1 traces
def _trace_golden():
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    g = np.load(os.path.join(here, "trace.npz"))
    blob = open(os.path.join(here, "trace_small.moepa"), "rb").read()
    ties = open(os.path.join(here, "trace_ties.moepa"), "rb").read()
    return g, blob, ties


def test_oracle_trace_reads_reference_files():
    from oracle import trace as T
    g, blob, ties = _trace_golden()
    d, e, k, acts, scores, topk = T.read_trace(blob)
    assert [d, e, k, len(acts)] == g["dims"].tolist()
    assert np.array_equal(acts, g["acts"]) and np.array_equal(scores, g["scores"])
    assert np.array_equal(topk, g["topk"])
    assert np.array_equal(T.read_trace(ties)[5], g["tie_topk"])


def test_oracle_trace_corruptions_match_reference_exceptions():
    from trace_corrupt import corruptions
    from oracle import trace as T
    g, blob, _ = _trace_golden()
    d, e, k, _n = g["dims"].tolist()
    bad = corruptions(blob, d, e, k)
    for name, kind, msg in zip(g["corrupt_names"], g["corrupt_kinds"], g["corrupt_msgs"]):
        with pytest.raises(T.OracleTraceError) as ei:
            T.read_trace(bad[str(name)])
        assert ei.value.kind == kind and str(ei.value) == msg, name
