"""GPU parity of the training path: labels (K3) and all loss families (K4)
against the reference goldens, fp64 backward (K5 + fp64 GEMM) and optimizer
(K6), a whole fp64 train() against the oracle's restated loop, and the fp32
tensor-core mode within its stated tolerance."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2511_10676_b200 as pb
    return pb


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    return oracle


def test_labels_and_losses_golden(pb, golden):
    g = golden("losses")
    for n, e, k in ((4, 8, 2), (16, 16, 2), (8, 64, 6)):
        pre = f"n{n}e{e}k{k}_"
        lab = pb.BatchLabels.from_scores(g[pre + "scores"], k)
        assert np.array_equal(lab.rank_of, g[pre + "rank_of"])
        assert np.array_equal(lab.topk_mask, g[pre + "mask"])
        for fam in ("mse", "wbce", "focal", "ranking"):
            loss, grad = pb.loss_and_grad(pb.LossSpec(family=fam), g[pre + "z"], lab)
            assert loss == pytest.approx(float(g[pre + fam + "_loss"]), rel=1e-12, abs=1e-15), fam
            assert np.allclose(grad, g[pre + fam + "_grad"], rtol=1e-10, atol=1e-15), fam
        _, _, n_pairs = pb.ranking_hinge(g[pre + "z"], lab)
        assert n_pairs == int(g[pre + "n_pairs"])


def test_loss_known_answers(pb):
    lab = pb.BatchLabels.from_scores(np.array([[0.9, 0.1]]), 1)
    loss, _ = pb.weighted_bce_loss(np.zeros((1, 2)), lab)
    assert loss == pytest.approx(3.0 * np.log(2.0), abs=1e-12)  # test_losses.py:78-83
    lab = pb.BatchLabels.from_scores(np.array([[0.7, 0.3]]), 1)
    h, _, n_pairs = pb.ranking_hinge(np.ones((1, 2)), lab, margin=0.1)
    assert n_pairs == 1 and h == pytest.approx(0.1)  # test_losses.py:133-137
    lab = pb.BatchLabels(np.array([[0.4, 0.4, 0.2]]), np.array([[True, True, False]]), np.array([[1, 2, 3]]))
    assert pb.ranking_hinge(np.zeros((1, 3)), lab)[2] == 2  # tie exclusion, test_losses.py:159-168


def test_backward_golden_arch2(pb, golden):
    g = golden("predictor")
    pre = "small_arch2_"
    m = pb.PredictorModel("arch2", g[pre + "w1"], g[pre + "b1"], g[pre + "w2"], g[pre + "b2"])
    grads = pb.backward(m, g[pre + "x"], g[pre + "dz"])
    for name in ("w1", "b1", "w2", "b2"):
        assert np.allclose(grads[name], g[pre + "grad_" + name], rtol=1e-10, atol=1e-12), name


def test_train_forward_backward_paired(pb, rng):
    m = pb.init_model("arch2", 8, 16, 8, seed=7)
    m.train()
    x = rng.standard_normal((4, 8))
    with pytest.raises(pb.UsageError):
        pb.backward(m, x, np.ones((4, 8)))
    pb.forward(m, x)
    with pytest.raises(pb.UsageError):
        pb.backward(m, rng.standard_normal((4, 8)), np.ones((4, 8)))
    g = pb.backward(m, x, np.zeros((4, 8)))
    assert all(np.all(v == 0) for v in g.values())


def test_optimizer_golden(pb, golden):
    from paper_2511_10676_b200 import _lib
    g = golden("optim")
    for opt, lr, kind in (("adam", 1e-3, 2), ("sgd", 0.05, 0), ("momentum", 0.02, 1)):
        p = torch.as_tensor(np.concatenate([g["p0_w"].ravel(), g["p0_b"]])).cuda()
        m = torch.zeros_like(p)
        v = torch.zeros_like(p)
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        for t in range(3):
            gr = torch.as_tensor(np.concatenate([g[f"{opt}_g{t}_w"].ravel(), g[f"{opt}_g{t}_b"]])).cuda()
            a = _lib.OptimArgs()
            a.kind, a.dtype, a.n = kind, _lib.MOEP_F64, p.numel()
            a.params, a.grads, a.m, a.v = p.data_ptr(), gr.data_ptr(), m.data_ptr(), v.data_ptr()
            a.lr, a.beta1, a.beta2, a.eps, a.momentum, a.t = lr, 0.9, 0.999, 1e-8, 0.9, t + 1
            a.shadow_bf16, a.n_shadow, a.nonfinite = None, 0, bad.data_ptr()
            _lib.check(_lib.lib().moep_optim_step(a, torch.cuda.current_stream().cuda_stream), "optim")
        want = np.concatenate([g[f"{opt}_p3_w"].ravel(), g[f"{opt}_p3_b"]])
        assert np.allclose(p.cpu().numpy(), want, rtol=1e-14, atol=1e-15), opt


def _dataset(O, n=1200, d=16, e=8, k=2, seed=7):
    r = np.random.default_rng(seed)
    gate = r.standard_normal((e, d)) / 4.0
    x = r.standard_normal((n, d))
    scores = O.teacher_scores(x, gate).astype(np.float32)
    acts = x.astype(np.float32)
    topk = O.top_k_batch(scores.astype(np.float64), k)
    return acts, scores, topk


@pytest.mark.parametrize("family", ["wbce", "ranking", "focal", "mse"])
def test_train_fp64_matches_oracle_loop(pb, O, family):
    acts, scores, topk = _dataset(O)
    cfg = pb.TrainConfig(loss=pb.LossSpec(family=family), hidden=32, batch_size=64, epochs=2, seed=5,
                         eval_fraction=0.2, precision="fp64")
    data = pb.TraceFile(16, 8, 2, acts, scores, topk)
    model, report = pb.train(cfg, data)
    p, rows, _ = O.train_arch2(acts, scores, topk, 2, hidden=32, batch_size=64, epochs=2, seed=5,
                               eval_fraction=0.2, loss={"family": family})
    for name in ("w1", "b1", "w2", "b2"):
        assert np.allclose(getattr(model, name), p[name], rtol=1e-8, atol=1e-10), name
    for ours, ref in zip(report.epochs, rows):
        assert ours.train_loss == pytest.approx(ref[0], rel=1e-9)
        assert (ours.exact_match, ours.top1, ours.overprov) == pytest.approx(ref[1:], abs=0)


def test_backward_golden_arch1_eval(pb, golden):
    g = golden("predictor")
    pre = "small_arch1_"
    m = pb.PredictorModel("arch1", g[pre + "w1"], g[pre + "b1"], g[pre + "w2"], g[pre + "b2"],
                          **{n: g[pre + n] for n in ("bn_scale", "bn_shift", "bn_mean", "bn_var")})
    grads = pb.backward(m, g[pre + "x"], g[pre + "dz"])
    for name in ("w1", "b1", "w2", "b2", "bn_scale", "bn_shift"):
        assert np.allclose(grads[name], g[pre + "grad_" + name], rtol=1e-10, atol=1e-12), name


def _perturbed_arch1(pb, rng):
    m = pb.init_model("arch1", 8, 16, 8, seed=7)
    for p in m.param_dict().values():
        p += 0.3 * rng.standard_normal(p.shape)
    m.bn_mean += 0.1 * rng.standard_normal(16)
    m.bn_var = np.abs(m.bn_var + 0.2 * rng.standard_normal(16))
    return m


def _oracle_params(m):
    return {"arch": "arch1", "w1": m.w1.copy(), "b1": m.b1.copy(), "w2": m.w2.copy(), "b2": m.b2.copy(),
            "bn_scale": m.bn_scale.copy(), "bn_shift": m.bn_shift.copy(), "bn_mean": m.bn_mean.copy(),
            "bn_var": m.bn_var.copy(), "bn_eps": m.bn_eps}


def test_arch1_train_forward_backward_vs_oracle(pb, O, rng):
    """BN batch statistics, running update, Philox dropout stream and the BN-train backward."""
    m = _perturbed_arch1(pb, rng)
    p = _oracle_params(m)
    state = {"seed": m.dropout_seed, "step": 0}
    m.train()
    x = rng.standard_normal((12, 8))
    for step in range(3):  # consecutive forwards draw consecutive dropout masks
        z = pb.forward(m, x)
        zr, cache = O.forward_train_arch1(p, x, state)
        assert np.allclose(z, zr, rtol=1e-11, atol=1e-12), step
        assert np.allclose(m.bn_mean, p["bn_mean"], rtol=1e-13, atol=1e-15)
        assert np.allclose(m.bn_var, p["bn_var"], rtol=1e-13, atol=1e-15)
        assert m._dropout_step == state["step"]
    dz = rng.standard_normal(z.shape)
    g = pb.backward(m, x, dz)
    gr = O.backward_train_arch1(p, cache, dz)
    for name in ("w1", "b1", "w2", "b2", "bn_scale", "bn_shift"):
        assert np.allclose(g[name], gr[name], rtol=1e-9, atol=1e-12), name
    # a supplied mask is used verbatim (predictor.py:243-245)
    mask = rng.random((12, 16)) >= 0.1
    z = pb.forward(m, x, dropout_mask=mask)
    zr, _ = O.forward_train_arch1(p, x, state, dropout_mask=mask)
    assert np.allclose(z, zr, rtol=1e-11, atol=1e-12)


def test_train_arch1_fp64_matches_oracle_loop(pb, O):
    acts, scores, topk = _dataset(O, n=600)
    cfg = pb.TrainConfig(loss=pb.LossSpec(family="ranking"), arch="arch1", hidden=32, batch_size=64, epochs=2,
                         seed=3, eval_fraction=0.2, precision="fp64")
    model, report = pb.train(cfg, pb.TraceFile(16, 8, 2, acts, scores, topk))
    p, rows, _ = O.train_arch2(acts, scores, topk, 2, hidden=32, batch_size=64, epochs=2, seed=3,
                               eval_fraction=0.2, loss={"family": "ranking"}, arch="arch1")
    for name in ("w1", "b1", "w2", "b2", "bn_scale", "bn_shift", "bn_mean", "bn_var"):
        assert np.allclose(getattr(model, name), p[name], rtol=1e-8, atol=1e-10), name
    for ours, ref in zip(report.epochs, rows):
        assert ours.train_loss == pytest.approx(ref[0], rel=1e-9)
        assert (ours.exact_match, ours.top1, ours.overprov) == pytest.approx(ref[1:], abs=0)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_train_c4_shape_fp32_step_within_tolerance(pb, O, precision):
    """Phi-mini shape (d=4096, h=2048, E=16, k=2), arch2 + ranking, one tensor-core
    step (fp32 master; tcgen05 dW1 on the hi/lo split or the bf16 dA) vs the
    fp64 oracle step: loss rel 1e-5; gradient norms rel 1e-4 (hi/lo: dA kept
    to 2^-16) or 5e-3 (bf16 dA: 2^-9 per element)."""
    r = np.random.default_rng(1)
    n, d, h, e, k = 256, 4096, 2048, 16, 2
    m = pb.init_model("arch2", d, h, e, seed=3)
    m.w1, m.w2 = O.round_bf16(m.w1), O.round_bf16(m.w2)
    x = O.round_bf16(r.standard_normal((n, d)))
    scores = O.teacher_scores(x, r.standard_normal((e, d)) / 64.0)
    spec = pb.LossSpec(family="ranking")
    tr = pb.DeviceTrainer(m, spec, "adam", 1e-3, precision=precision)
    lab = pb.BatchLabels.from_scores(torch.as_tensor(scores).cuda(), k)
    out = tr.step(torch.as_tensor(x).cuda().to(torch.bfloat16), lab.true_scores.float().contiguous(),
                  lab.topk_mask.to(torch.uint8).contiguous(), lab.rank_of.contiguous())
    p = {"arch": "arch2", "w1": m.w1.copy(), "b1": m.b1.copy(), "w2": m.w2.copy(), "b2": m.b2.copy()}
    z, cache = O.forward_eval(p, x)
    olab = O.batch_labels(scores, k)
    lv, dz = O.loss_and_grad({"family": "ranking"}, z, olab)
    g = O.backward_eval(p, cache, dz)
    assert float(out[0].item()) == pytest.approx(lv, rel=1e-5)
    tol = 1e-4 if precision == "fp32" else 5e-3
    gw1 = tr.view(tr.grad, 0).double().cpu().numpy()
    e1 = np.linalg.norm(gw1 - g["w1"]) / np.linalg.norm(g["w1"])
    assert e1 < tol, e1
    gw2 = tr.view(tr.grad, 1).double().cpu().numpy()
    e2 = np.linalg.norm(gw2 - g["w2"]) / np.linalg.norm(g["w2"])
    assert e2 < tol, e2


@pytest.mark.parametrize("n,h,d,passes", [(16384, 2048, 4096, 2), (16384, 2048, 4096, 1), (1000, 200, 136, 1),
                                          (323, 128, 256, 2), (4096, 384, 512, 2)])
def test_dw1_tcgen05_gemm(pb, n, h, d, passes):
    """moep_dw1_bf16 (tcgen05, MN-major TMA operands, K-split + fixed-order
    reduce) against an fp64 reference of sum_p dA_p^T X: the products are
    exact, the fp32 accumulation is the only error (rel 1e-5 of the norm)."""
    from paper_2511_10676_b200._lib import check, lib, ptr
    g = torch.Generator(device="cuda")
    g.manual_seed(n + h + d)
    da = torch.randn((n, passes * h), device="cuda", generator=g).to(torch.bfloat16)
    x = torch.randn((n, d), device="cuda", generator=g).to(torch.bfloat16)
    out = torch.full((h, d), float("nan"), dtype=torch.float32, device="cuda")
    need = int(lib().moep_dw1_workspace_floats(h, d, n, passes))
    ws = torch.zeros(max(need, 1), dtype=torch.float32, device="cuda")
    check(lib().moep_dw1_bf16(ptr(da), ptr(x), n, h, d, passes, ptr(out), ptr(ws), need,
                              torch.cuda.current_stream().cuda_stream), "moep_dw1_bf16")
    ref = sum(da[:, p * h:(p + 1) * h].double().T @ x.double() for p in range(passes))
    err = float(torch.linalg.vector_norm(out.double() - ref) / torch.linalg.vector_norm(ref))
    assert err < 1e-5, err
    assert float((out.double() - ref).abs().max()) < 1e-4 * float(ref.abs().max()) + 1e-6


def test_train_nonfinite_guard_reports_first_step(pb, O):
    """The reference raises FloatingPointError at the first step whose loss or
    parameters are non-finite (trainer.py:125-128, 184-187); the device loop
    keeps a per-step flag and names the same step."""
    acts, scores, topk = _dataset(O)
    acts = acts.copy()
    cfg = pb.TrainConfig(loss=pb.LossSpec(family="wbce"), hidden=32, batch_size=64, epochs=1, seed=5,
                         eval_fraction=0.2, precision="fp64", learning_rate=1e300)
    with pytest.raises(FloatingPointError) as e1:
        pb.train(cfg, pb.TraceFile(16, 8, 2, acts, scores, topk))
    with pytest.raises(FloatingPointError) as e2:
        O.train_arch2(acts, scores, topk, 2, hidden=32, batch_size=64, epochs=1, seed=5, eval_fraction=0.2,
                      loss={"family": "wbce"}, lr=1e300)
    assert str(e1.value) == str(e2.value)
