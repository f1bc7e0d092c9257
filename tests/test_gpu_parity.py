"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference's golden fixtures. Bit-exact for ids / counters; predict_logits is
exact fp64 (fixed summation order, so within 1e-11 of numpy's BLAS order);
K1's raw fp32 logits (logits(approx=True)) within tau_rel/2 of the row scale
||h|| max_e||w2_e||, the margin contract of DESIGN §3."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

LOGIT_ATOL = 1e-11   # predict_logits (exact fp64, fixed order) vs numpy fp64 (BLAS order)


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


def bf16_model(pb, O, arch, d, h, e, seed, rng=None):
    m = pb.init_model(arch, d, h, e, seed=seed)
    m.w1 = O.round_bf16(m.w1)
    m.w2 = O.round_bf16(m.w2)
    if arch == "arch1" and rng is not None:
        m.bn_mean = rng.standard_normal(h) * 0.05
        m.bn_var = 0.3 + rng.random(h) * 0.5
        m.bn_scale = 1 + 0.1 * rng.standard_normal(h)
        m.bn_shift = 0.1 * rng.standard_normal(h)
    return m


def oracle_params(m):
    p = {"arch": m.arch, "w1": m.w1, "b1": m.b1, "w2": m.w2, "b2": m.b2}
    if m.arch == "arch1":
        p.update(bn_scale=m.bn_scale, bn_shift=m.bn_shift, bn_mean=m.bn_mean, bn_var=m.bn_var)
    return p


# ------------------------------------------------------------- goldens
@pytest.mark.parametrize("arch", ["arch1", "arch2"])
def test_small_reference_shapes_golden(pb, golden, arch):
    """d=8, h=16, E=8 perturbed models from the reference tests (fp64 weights -> K2 path)."""
    g = golden("predictor")
    pre = f"small_{arch}_"
    kw = {n: g[pre + n] for n in ("bn_scale", "bn_shift", "bn_mean", "bn_var")} if arch == "arch1" else {}
    m = pb.PredictorModel(arch, g[pre + "w1"], g[pre + "b1"], g[pre + "w2"], g[pre + "b2"], **kw)
    z = pb.predict_logits(m, g[pre + "x"])
    assert np.allclose(z, g[pre + "logits"], rtol=0, atol=1e-12)
    assert np.array_equal(pb.predict_topk_batch(m, g[pre + "x"], 3), g[pre + "top3"])


def test_c1_golden_ids(pb, golden, O):
    """bf16-representable C1 layer: K1 tensor-core path + fix-up equals the reference."""
    g = golden("predictor")
    m = bf16_model(pb, O, "arch2", 2048, 2048, 64, seed=0)
    x = g["c1_x"].astype(np.float64)
    assert np.array_equal(pb.predict_topk_batch(m, x, 6), g["c1_top6"])
    assert np.array_equal(pb.predict_topk_batch(m, x, 10), g["c1_top10"])
    z = pb.predict_logits(m, x)
    assert np.abs(z - g["c1_logits"]).max() < LOGIT_ATOL


def test_topk_golden(pb, golden):
    g = golden("topk")
    for k in (1, 3, 6, 11):
        assert np.array_equal(pb.top_k_batch(g["tie_scores"], k), g[f"tie_top{k}"])
    for k in (1, 6, 10, 64):
        assert np.array_equal(pb.top_k_batch(g["rand_scores"], k), g[f"rand_top{k}"])
    assert np.array_equal(pb.rank_order(g["rand_scores"]), g["rand_order"])


def test_topk_hand_cases(pb):
    # test_core.py:60-64, 78-79 + signed zero ties
    assert pb.top_k(np.array([0.1, 0.7, 0.2]), 1).tolist() == [1]
    assert pb.top_k(np.array([0.5, 0.5, 0.0]), 1).tolist() == [0]
    assert pb.top_k(np.array([0.4, 0.1, 0.3, 0.2]), 2).tolist() == [0, 2]
    assert pb.top_k(np.array([-0.0, 0.0, -1.0]), 1).tolist() == [0]
    with pytest.raises(ValueError):
        pb.top_k(np.array([1.0, 2.0]), 3)


def test_eval_logits_golden(pb, golden):
    from paper_2511_10676_b200.engine import EvalCounters, eval_logits_device
    g = golden("metrics")
    for idx in range(4):
        pre = f"m{idx}_"
        z, truth = g[pre + "z"], g[pre + "truth"]
        n, e = z.shape
        k = truth.shape[1]
        ms = g[pre + "m_list"].tolist()
        c = eval_logits_device(torch.from_numpy(z).cuda(), torch.from_numpy(truth), k, e, ms).cpu().numpy()
        ec = EvalCounters.from_array(c, k, e, ms)
        assert ec.overprov[k] / n == float(g[pre + "exact"])
        assert ec.top1 / n == float(g[pre + "top1"])
        assert [ec.overprov[m] / n for m in ms] == g[pre + "overprov"].tolist()
        assert [ec.recall[m] / (n * k) for m in ms] == g[pre + "recall"].tolist()
        assert np.array_equal(ec.per_expert_hits, g[pre + "hits"])
        assert np.array_equal(ec.per_expert_truth, g[pre + "truthc"])


# ---------------------------------------------- seeded parity vs the oracle
CONFIGS = [
    # (arch, d, h, E, k, n)    C1/C2 DSV2L, C3 Qwen3, C4 Phi (inference), arch1
    ("arch2", 2048, 2048, 64, 6, 16384),
    ("arch2", 2048, 2048, 128, 8, 8192),
    ("arch2", 2048, 2048, 128, 8, 20480),  # C3 Qwen3 with every CTA pair busy (unsplit, one wave: v2)
    # >= 2 tiles of 256 per CTA pair (N >= 37,888 on 148 SMs): the v4 kernel
    # (token epilogue on its own warpgroup, A2 in TMEM); ragged last tile
    ("arch2", 2048, 2048, 64, 6, 40000),
    ("arch2", 2048, 2048, 128, 8, 40000),
    ("arch2", 4096, 2048, 16, 2, 40000),
    ("arch1", 2048, 2048, 64, 6, 40000),
    ("arch2", 4096, 2048, 16, 2, 8192),
    ("arch1", 2048, 2048, 64, 6, 4096),
    ("arch2", 64, 128, 16, 2, 3000),     # ragged token count, small dims
    ("arch2", 8, 16, 8, 2, 257),         # reference test dims through the tensor-core path
]


@pytest.mark.parametrize("arch,d,h,e,k,n", CONFIGS)
def test_k1_ids_and_counters_vs_oracle(pb, O, arch, d, h, e, k, n):
    rng = np.random.default_rng(d * 7 + e)
    m = bf16_model(pb, O, arch, d, h, e, seed=3, rng=rng)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref = O.predict_logits(oracle_params(m), x)
    dev = m.to_device()
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    assert dev.k1_usable(True, (k,))
    for mm in sorted({1, k, min(k + 4, e)}):
        if mm <= 15 or mm == e:
            ids, flags = dev.topk(xt, mm, return_flags=True)
            assert np.array_equal(ids.cpu().numpy(), O.top_k_batch(zref, mm)), mm
    z = dev.logits(xt).cpu().numpy()
    assert np.abs(z - zref).max() < LOGIT_ATOL
    truth = O.top_k_batch(zref + 0.05 * rng.standard_normal(zref.shape), k)  # correlated truth
    ms = O.default_m_list(k, e)
    cnt, fcount, _ = dev.evaluate(xt, torch.from_numpy(truth), k, ms)
    c = pb.EvalCounters.from_array(cnt.cpu().numpy(), k, e, sorted(set(ms) | {k}))
    oc = O.eval_counters(zref, truth, e, ms)
    assert c.n == oc["n"] and c.top1 == oc["top1_count"]
    assert c.overprov == oc["overprov_count"] and c.recall == oc["recall_count"]
    assert np.array_equal(c.per_expert_hits, oc["per_expert_hits"])
    assert np.array_equal(c.per_expert_truth, oc["per_expert_truth"])


@pytest.mark.parametrize("n,e,kernel", [(16384, 64, 2), (40000, 64, 4), (65536, 128, 4), (40000, 16, 4),
                                        (4096, 32, 1), (40000, 64, 5), (30000, 32, 5), (20000, 16, 5)])
def test_margin_covers_error(pb, O, n, e, kernel):
    """Calibration guard: K1's raw error / row scale stays 4x inside the margin
    (max <= tau/4; tau/2 is the hard limit) on each kernel: v2 (one wave), v4
    (>= 2 tiles per CTA pair; E = 128 has no separate lo accumulator and runs
    with 1.5 tau), v5 (4-CTA clusters, partial logits of two pairs summed) and
    the 1-SM kernel."""
    from paper_2511_10676_b200 import _lib
    from paper_2511_10676_b200.engine import TAU_REL
    rng = np.random.default_rng(11 + e)
    d = h = 2048 if kernel != 1 else 512
    if kernel == 1:
        h = 384
    m = bf16_model(pb, O, "arch2", d, h, e, seed=5)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref, cache = O.forward_eval(oracle_params(m), x)
    dev = m.to_device()
    lg = torch.empty((n, e), dtype=torch.float32, device="cuda")
    dev._k1(torch.from_numpy(x).to("cuda", torch.bfloat16), logits=lg, kernel=kernel)
    err = np.abs(lg.double().cpu().numpy() - zref).max(axis=1)
    scale = np.linalg.norm(cache["h"], axis=1) * np.linalg.norm(m.w2, axis=1).max()
    ratio = err / scale
    tau = TAU_REL * (1.5 if (kernel == 4 and e > 64) or kernel == 1 else 1.0)
    assert 4 * ratio.max() <= tau, (ratio.max(), tau)


@pytest.mark.parametrize("n,e", [(256, 64), (4096, 64), (8192, 128), (300, 16)])
def test_margin_covers_error_hidden_split(pb, O, n, e):
    """Same guard for the hidden-split K1 (small N: partial logits per hidden
    group summed in fp32 by the finish kernel), and the split path equals the
    unsplit one on ids."""
    from paper_2511_10676_b200 import _lib
    from paper_2511_10676_b200.engine import TAU_REL
    d = h = 2048
    assert _lib.lib().moep_predict_split_floats(n, h, e) > 0
    rng = np.random.default_rng(n + e)
    m = bf16_model(pb, O, "arch2", d, h, e, seed=6)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref, cache = O.forward_eval(oracle_params(m), x)
    dev = m.to_device()
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    lg = torch.empty((n, e), dtype=torch.float32, device="cuda")
    dev._k1(xt, logits=lg)
    err = np.abs(lg.double().cpu().numpy() - zref).max(axis=1)
    scale = np.linalg.norm(cache["h"], axis=1) * np.linalg.norm(m.w2, axis=1).max()
    assert 4 * (err / scale).max() <= TAU_REL, (err / scale).max()
    dev.decode_max_tokens = 0
    ids_split = dev.topk(xt, 6).cpu().numpy()
    dev.split_hidden = False
    ids_flat = dev.topk(xt, 6).cpu().numpy()
    assert np.array_equal(ids_split, O.top_k_batch(zref, 6))
    assert np.array_equal(ids_split, ids_flat)


def test_ties_go_to_fp64_and_lower_index(pb, O):
    """Duplicate W2 rows give exact logit ties; the lower expert index must win."""
    rng = np.random.default_rng(3)
    m = bf16_model(pb, O, "arch2", 256, 256, 16, seed=9)
    m.w2[5] = m.w2[2]
    m.w2[9] = m.w2[2]
    x = O.round_bf16(rng.standard_normal((512, 256)))
    zref = O.predict_logits(oracle_params(m), x)
    for mm in (1, 2, 3, 4):
        assert np.array_equal(pb.predict_topk_batch(m, x, mm), O.top_k_batch(zref, mm))


def test_eval_margin_flags_only_true_expert_ties(pb, O):
    """Evaluation-only boundaries (no ids output): an exact logit tie between
    experts 2 and 5 can only change the counters when a TRUE expert sits in the
    tie window. With truth sets that avoid both, no token is flagged yet every
    counter equals the oracle's; with truth sets that contain them, the tied
    tokens are flagged, recomputed in fp64, and the counters still match."""
    rng = np.random.default_rng(17)
    e, k = 16, 2
    m = bf16_model(pb, O, "arch2", 256, 256, e, seed=4)
    m.w2[5] = m.w2[2]
    x = O.round_bf16(rng.standard_normal((4096, 256)))
    zref = O.predict_logits(oracle_params(m), x)
    dev = m.to_device()
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    ms = [2, 6, 16]
    others = np.array([i for i in range(e) if i not in (2, 5)])
    t_avoid = np.sort(np.stack([rng.choice(others, k, replace=False) for _ in range(len(x))]), axis=1)
    t_hit = np.sort(np.stack([np.array([2, rng.choice(others)]) for _ in range(len(x))]), axis=1)
    for truth, expect_flags in ((t_avoid, False), (t_hit, True)):
        cnt, fcount, _ = dev.evaluate(xt, torch.from_numpy(truth), k, ms)
        c = pb.EvalCounters.from_array(cnt.cpu().numpy(), k, e, ms)
        oc = O.eval_counters(zref, truth, e, ms)
        assert c.top1 == oc["top1_count"] and c.overprov == oc["overprov_count"] and c.recall == oc["recall_count"]
        assert np.array_equal(c.per_expert_hits, oc["per_expert_hits"])
        nflag = int(fcount.item())
        assert (nflag > 0) == expect_flags, nflag


def test_nonfinite_input_raises(pb, O):
    m = bf16_model(pb, O, "arch2", 64, 128, 16, seed=1)
    x = np.zeros((4, 64))
    x[2, 3] = np.nan
    with pytest.raises(pb.ConfigurationError):
        pb.predict_logits(m, x)
    with pytest.raises(pb.ConfigurationError):
        pb.predict_logits(m, np.zeros((4, 65)))


@pytest.mark.parametrize("n", [3000, 40000])
def test_nonfinite_bf16_input_raises_through_k1_status(pb, O, n):
    """bf16 device input takes K1 with no isfinite pass: a NaN / Inf token makes
    its fp32 logits non-finite, K1 sets its status word and the API raises the
    reference's ConfigurationError (predictor.py:188-189). With the caller's own
    status word nothing synchronises; check_status raises afterwards."""
    rng = np.random.default_rng(4)
    m = bf16_model(pb, O, "arch2", 512, 512, 64, seed=1)
    dev = m.to_device()
    dev.decode_max_tokens = 0
    x = torch.from_numpy(O.round_bf16(rng.standard_normal((n, 512)))).to("cuda", torch.bfloat16)
    truth = torch.from_numpy(O.top_k_batch(rng.standard_normal((n, 64)), 6))
    st = dev.new_status()
    dev.topk(x, 6, status=st)
    dev.evaluate(x, truth, 6, [6, 10, 64], ids_m=6, status=st)
    assert int(st.item()) == 0
    dev.check_status(st, x)
    for bad in (float("nan"), float("inf")):
        xb = x.clone()
        xb[n // 2, 7] = bad
        with pytest.raises(pb.ConfigurationError):
            dev.topk(xb, 6)
        with pytest.raises(pb.ConfigurationError):
            dev.evaluate(xb, truth, 6, [6, 10, 64])
        st = dev.new_status()
        dev.evaluate(xb, truth, 6, [6, 10, 64], ids_m=6, status=st)
        assert int(st.item()) & 1
        with pytest.raises(pb.ConfigurationError):
            dev.check_status(st, xb)


def test_large_biases_in_margin(pb, O):
    """Biases far above the logit scale: K1 holds b1 / b2 in fp32,
    so the margin adds 2^-21 (max|b2| + 1.2 max||w2_e|| ||b1||); ids and
    counters must still equal the oracle's."""
    rng = np.random.default_rng(31)
    n, d, h, e, k = 40000, 2048, 2048, 64, 6
    m = bf16_model(pb, O, "arch2", d, h, e, seed=8)
    m.b2 = 200.0 + 0.02 * rng.standard_normal(e)   # logits ~ N(0, 0.18) on top of ~200
    m.b1 = 3.0 * rng.standard_normal(h)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref = O.predict_logits(oracle_params(m), x)
    dev = m.to_device()
    assert dev.tau_bias > 0
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    for mm in (1, 6, 10):
        assert np.array_equal(dev.topk(xt, mm).cpu().numpy(), O.top_k_batch(zref, mm)), mm
    truth = O.top_k_batch(zref + 0.05 * rng.standard_normal(zref.shape), k)
    cnt, _, ids = dev.evaluate(xt, torch.from_numpy(truth), k, [6, 10, 64], ids_m=6)
    c = pb.EvalCounters.from_array(cnt.cpu().numpy(), k, e, [6, 10, 64])
    oc = O.eval_counters(zref, truth, e, [6, 10, 64])
    assert c.overprov == oc["overprov_count"] and c.recall == oc["recall_count"] and c.top1 == oc["top1_count"]
    assert np.array_equal(ids.cpu().numpy(), O.top_k_batch(zref, 6))


def test_forced_kernels_agree(pb, O):
    """The four K1 kernels (1-SM, pair v2, pair v4, cluster v5;
    moep_predict_args.kernel) give identical ids on the same input after the fix-up."""
    rng = np.random.default_rng(12)
    n, d, h, e = 40000, 1024, 1024, 64
    m = bf16_model(pb, O, "arch2", d, h, e, seed=12)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref = O.predict_logits(oracle_params(m), x)
    ref = O.top_k_batch(zref, 6)
    dev = m.to_device()
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    from paper_2511_10676_b200.engine import MOEP_BF16
    for kern in (1, 2, 4, 5):
        ids = torch.empty((n, 6), dtype=torch.int32, device="cuda")
        flags, flist, fcount = dev._k1(xt, m_sel=6, bounds=(6,), ids=ids, kernel=kern)
        a = dev._fp64_args(xt, MOEP_BF16, rows=flist, row_count=fcount, m_sel=6, ids=ids)
        dev._fixup(a, n)
        assert np.array_equal(ids.cpu().numpy(), ref), kern


def test_logits_exact_and_approx(pb, O):
    """predict_logits returns exact fp64 for every row; the opt-in
    approx=True returns K1's fp32 logits, each within tau/2 of the row scale."""
    rng = np.random.default_rng(19)
    n, d, h, e = 5000, 2048, 2048, 64
    m = bf16_model(pb, O, "arch2", d, h, e, seed=2)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref, cache = O.forward_eval(oracle_params(m), x)
    dev = m.to_device()
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    assert np.allclose(dev.logits(xt).cpu().numpy(), zref, rtol=0, atol=LOGIT_ATOL)
    assert np.allclose(pb.predict_logits(m, x), zref, rtol=0, atol=LOGIT_ATOL)
    za = dev.logits(xt, approx=True).cpu().numpy()
    scale = np.linalg.norm(cache["h"], axis=1) * np.linalg.norm(m.w2, axis=1).max()
    assert (np.abs(za - zref).max(axis=1) <= dev.tau_rel / 2 * scale + dev.tau_abs).all()


def test_single_vector_and_m_range(pb, O):
    m = bf16_model(pb, O, "arch2", 64, 128, 16, seed=1)
    x = O.round_bf16(np.random.default_rng(0).standard_normal(64))
    z = pb.predict_logits(m, x)
    assert z.shape == (16,)
    sel = pb.predict_topk(m, x, 4)
    assert sel.indices.tolist() == O.top_k(O.predict_logits(oracle_params(m), x[None])[0], 4).tolist()
    with pytest.raises(ValueError):
        pb.predict_topk_batch(m, x[None], 17)
    m.train()
    with pytest.raises(pb.UsageError):
        pb.predict_topk(m, x, 1)


def test_non_bf16_inputs_take_exact_fp64_path(pb, O):
    rng = np.random.default_rng(2)
    m = pb.init_model("arch2", 64, 96, 16, seed=4)  # fp64 weights, not bf16-representable
    x = rng.standard_normal((300, 64))
    zref = O.predict_logits(oracle_params(m), x)
    assert np.allclose(pb.predict_logits(m, x), zref, rtol=0, atol=1e-12)
    for mm in (1, 2, 7, 16):
        assert np.array_equal(pb.predict_topk_batch(m, x, mm), O.top_k_batch(zref, mm))


def test_input_norm_kernel(pb, O):
    rng = np.random.default_rng(5)
    x = 3 * rng.standard_normal((64, 2048)) + 0.5
    gamma = rng.uniform(0.5, 1.5, 2048)
    beta = 0.1 * rng.standard_normal(2048)
    m = bf16_model(pb, O, "arch2", 2048, 2048, 64, seed=0)
    dev = m.to_device()
    xt = torch.from_numpy(x).cuda()
    for kind, g, b in (("rmsnorm", gamma, None), ("layernorm", gamma, beta), ("layernorm", None, None)):
        out = dev.normalize(xt, kind, g, b).double().cpu().numpy()
        ref = O.input_norm_bf16(x, kind, g, b)
        assert np.array_equal(out, ref), kind


@pytest.mark.parametrize("tau_rel,lo,hi", [(1e-3, 513, 3000), (1.5e-5, 1, 512)])
def test_fixup_overflow_path(pb, O, tau_rel, lo, hi):
    """Flagged rows beyond the fix-up capacity go through the per-group fp64
    kernel; results must be identical either way (forced tiny capacity + a wide
    margin). The two margins put the flagged count on either side of the
    device-side switch between the split-hidden and the GEMM fix-up kernels."""
    rng = np.random.default_rng(21)
    m = bf16_model(pb, O, "arch2", 512, 512, 64, seed=2)
    x = O.round_bf16(rng.standard_normal((3000, 512)))
    zref = O.predict_logits(oracle_params(m), x)
    truth = O.top_k_batch(zref + 0.05 * rng.standard_normal(zref.shape), 6)
    ms = [6, 10, 64]
    oc = O.eval_counters(zref, truth, 64, ms)
    for cap in (None, 8, 4096):
        dev = m.to_device(tau_rel=tau_rel)
        dev.fixup_capacity = cap
        xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
        assert np.array_equal(dev.topk(xt, 6).cpu().numpy(), O.top_k_batch(zref, 6))
        cnt, fcount, _ = dev.evaluate(xt, torch.from_numpy(truth), 6, ms)
        assert lo <= int(fcount.item()) <= hi, int(fcount.item())
        c = pb.EvalCounters.from_array(cnt.cpu().numpy(), 6, 64, ms)
        assert c.overprov == oc["overprov_count"] and c.recall == oc["recall_count"]
        assert c.top1 == oc["top1_count"] and np.array_equal(c.per_expert_hits, oc["per_expert_hits"])
        z = dev.logits(xt).cpu().numpy()
        assert np.abs(z - zref).max() < LOGIT_ATOL


# ------------------------------------------------ shape / argument edge cases
EDGE = [
    # arch, d, h, E, k, n, ms        why
    ("arch2", 512, 512, 48, 6, 2000, (6, 10, 48)),     # E not a power of two (EP = 64 padding)
    ("arch2", 256, 384, 32, 4, 1500, (4, 8, 32)),      # hidden % 256 != 0 -> 1-SM kernel
    ("arch2", 512, 512, 64, 16, 1200, (15, 16, 64)),   # k = 16 (max truth) and m = 15 (max selection)
    ("arch1", 512, 512, 64, 6, 700, (6, 10, 64)),      # arch1 through the hidden split (small N)
    ("arch2", 136, 256, 16, 2, 333, (2, 6, 16)),       # d not a multiple of 64 (TMA tail K block)
]


@pytest.mark.parametrize("arch,d,h,e,k,n,ms", EDGE)
def test_edge_shapes_vs_oracle(pb, O, arch, d, h, e, k, n, ms):
    rng = np.random.default_rng(d + h + e + n)
    m = bf16_model(pb, O, arch, d, h, e, seed=11, rng=rng)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref = O.predict_logits(oracle_params(m), x)
    dev = m.to_device()
    dev.decode_max_tokens = 0
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    for mm in sorted({1, min(k, 15), 15 if e > 15 else e, e}):
        assert np.array_equal(dev.topk(xt, mm).cpu().numpy(), O.top_k_batch(zref, mm)), mm
    truth = O.top_k_batch(zref + 0.05 * rng.standard_normal(zref.shape), k)
    cnt, _, ids = dev.evaluate(xt, torch.from_numpy(truth), k, list(ms), ids_m=min(k, 15))
    c = pb.EvalCounters.from_array(cnt.cpu().numpy(), k, e, sorted(set(ms) | {k}))
    oc = O.eval_counters(zref, truth, e, list(ms))
    assert c.n == n and c.top1 == oc["top1_count"]
    assert c.overprov == oc["overprov_count"] and c.recall == oc["recall_count"]
    assert np.array_equal(c.per_expert_hits, oc["per_expert_hits"])
    assert np.array_equal(c.per_expert_truth, oc["per_expert_truth"])
    assert np.array_equal(ids.cpu().numpy(), O.top_k_batch(zref, min(k, 15)))


def test_ties_through_hidden_split_and_decode(pb, O):
    """Exact ties (duplicated W2 rows) on the split-hidden tensor path (N=300) and
    the decode path (N=5): lower index wins, as core.py:27-48."""
    rng = np.random.default_rng(8)
    m = bf16_model(pb, O, "arch2", 512, 512, 16, seed=4)
    m.w2[7] = m.w2[3]
    m.w2[12] = m.w2[3]
    for n in (300, 5):
        x = O.round_bf16(rng.standard_normal((n, 512)))
        zref = O.predict_logits(oracle_params(m), x)
        dev = m.to_device()
        xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
        for mm in (1, 2, 3, 5):
            assert np.array_equal(dev.topk(xt, mm).cpu().numpy(), O.top_k_batch(zref, mm)), (n, mm)


@pytest.mark.parametrize("n,e,arch", [(40000, 64, "arch2"), (33000, 32, "arch1"), (300, 64, "arch2"),
                                      (70001, 16, "arch2")])
def test_v5_cluster_kernel_evaluate(pb, O, n, e, arch):
    """K1 v5 (two CTA pairs per 256-token tile, x multicast, partial logits
    exchanged through distributed shared memory) through the full evaluate
    pipeline: ids and every counter equal the oracle's, including a ragged last
    tile, fewer tiles than clusters (n = 300) and arch1's activation."""
    rng = np.random.default_rng(n + e)
    d, h = 1024, 1536
    m = bf16_model(pb, O, arch, d, h, e, seed=9)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref = O.predict_logits(oracle_params(m), x)
    truth = O.top_k_batch(zref + 0.05 * rng.standard_normal(zref.shape), 6)
    dev = m.to_device()
    dev.k1_kernel = 5
    dev.decode_max_tokens = 0
    ms = [6, 10, e]
    cnt, fc, ids = dev.evaluate(torch.from_numpy(x).to("cuda", torch.bfloat16), torch.from_numpy(truth), 6, ms,
                                ids_m=6)
    assert np.array_equal(ids.cpu().numpy(), O.top_k_batch(zref, 6))
    c = pb.EvalCounters.from_array(cnt.cpu().numpy(), 6, e, ms)
    oc = O.eval_counters(zref, truth, e, ms)
    assert c.n == oc["n"] and c.top1 == oc["top1_count"]
    assert c.overprov == oc["overprov_count"] and c.recall == oc["recall_count"]
    assert np.array_equal(c.per_expert_hits, oc["per_expert_hits"])
    assert np.array_equal(c.per_expert_truth, oc["per_expert_truth"])


@pytest.mark.parametrize("e,k", [(128, 8), (16, 2)])
def test_v2_token_epilogue_staging_race(pb, O, e, k):
    """K1 v2 stages each token's logits in the A2 shared-memory region, whose
    per-warp A2 rows overlap OTHER warps' staging rows: a warp that finished
    its (data-dependent) selection must not write the next chunk's A2 while
    another still reads its staging row (found as a rare counter mismatch in a
    full-suite run; fixed with a warpgroup barrier). Repeated evaluations with
    truth-heavy windows must all equal the oracle."""
    rng = np.random.default_rng(4242 + e)
    n, d, h = 20480, 1024, 1024
    m = bf16_model(pb, O, "arch2", d, h, e, seed=8)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref = O.predict_logits(oracle_params(m), x)
    truth = O.top_k_batch(zref + 0.02 * rng.standard_normal(zref.shape), k)
    ms = O.default_m_list(k, e)
    oc = O.eval_counters(zref, truth, e, ms)
    dev = m.to_device()
    dev.k1_kernel = 2
    dev.decode_max_tokens = 0
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    tt = torch.from_numpy(truth)
    for _ in range(6):
        cnt, _, _ = dev.evaluate(xt, tt, k, ms)
        c = pb.EvalCounters.from_array(cnt.cpu().numpy(), k, e, sorted(set(ms) | {k}))
        assert c.n == oc["n"] and c.top1 == oc["top1_count"]
        assert c.overprov == oc["overprov_count"] and c.recall == oc["recall_count"]
        assert np.array_equal(c.per_expert_hits, oc["per_expert_hits"])


@pytest.mark.parametrize("arch,d,h,e,n", [("arch2", 2048, 2048, 64, 40000), ("arch2", 2048, 2048, 128, 20480),
                                          ("arch2", 1024, 1024, 16, 300), ("arch1", 1024, 1024, 32, 5000),
                                          ("arch2", 256, 384, 32, 2000)])
def test_fused_softmax_probs(pb, O, arch, d, h, e, n):
    """north_star (1)'s softmax stage: K1's fused softmax of its fp32 logits
    (core.softmax, core.py:19-24) against softmax of the exact fp64 logits.
    Each logit is within delta/2 of exact (the margin contract), so
    |p - p_ref| <= p_ref (exp(delta) - 1 + 1e-5) + 2^-22 per row, where the
    1e-5 covers the fp32 exp / sum / divide; rows sum to 1 within 1e-5.
    Covers v4, v2 (one wave), the hidden split, arch1 and the 1-SM kernel."""
    rng = np.random.default_rng(n + e)
    m = bf16_model(pb, O, arch, d, h, e, seed=21, rng=rng)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref, cache = O.forward_eval(oracle_params(m), x)
    dev = m.to_device()
    p = dev.probs(torch.from_numpy(x).to("cuda", torch.bfloat16)).double().cpu().numpy()
    pref = O.softmax(zref, axis=1)
    hn = np.linalg.norm(cache["h"], axis=1)
    delta = dev.tau_abs + dev.tau_bias + dev.tau_rel * (1.5 if e > 64 else 1.0) * hn * dev.w2_norm
    bound = pref * (np.expm1(delta)[:, None] + 1e-5) + 2.0 ** -22
    assert (np.abs(p - pref) <= bound).all(), np.abs(p - pref).max()
    assert np.allclose(p.sum(axis=1), 1.0, rtol=0, atol=1e-5)


@pytest.mark.parametrize("e,k", [(64, 6), (128, 8), (32, 4)])
def test_network_selection_ties_and_near_ties(pb, O, e, k):
    """K1's token selection (packed-key bitonic network) at v4 scale with
    exact ties (duplicate W2 rows) and near-ties (W2 rows one bf16 ulp apart
    in one element: logits equal in their top bits but distinct): those rows
    take the exact argmax path; ids and every counter equal the oracle's."""
    rng = np.random.default_rng(77 + e)
    n, d, h = 40000, 1024, 1024
    m = bf16_model(pb, O, "arch2", d, h, e, seed=13)
    m.w2[5] = m.w2[2]
    m.w2[9] = m.w2[2]
    m.w2[11] = m.w2[3].copy()
    j = int(np.argmax(np.abs(m.w2[11])))
    # one bf16 ulp up in one element (stays bf16-exact)
    mant, ex = np.frexp(m.w2[11, j])
    m.w2[11, j] = np.ldexp(mant + np.sign(mant) / 256.0, ex)
    assert np.array_equal(O.round_bf16(m.w2), m.w2)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref = O.predict_logits(oracle_params(m), x)
    truth = O.top_k_batch(zref + 0.01 * rng.standard_normal(zref.shape), k)
    ms = O.default_m_list(k, e)
    oc = O.eval_counters(zref, truth, e, ms)
    dev = m.to_device()
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    for mm in (1, k, k + 2):
        assert np.array_equal(dev.topk(xt, mm).cpu().numpy(), O.top_k_batch(zref, mm)), mm
    cnt, _, ids = dev.evaluate(xt, torch.from_numpy(truth), k, ms, ids_m=k)
    assert np.array_equal(ids.cpu().numpy(), O.top_k_batch(zref, k))
    c = pb.EvalCounters.from_array(cnt.cpu().numpy(), k, e, sorted(set(ms) | {k}))
    assert c.n == oc["n"] and c.top1 == oc["top1_count"]
    assert c.overprov == oc["overprov_count"] and c.recall == oc["recall_count"]
    assert np.array_equal(c.per_expert_hits, oc["per_expert_hits"])
