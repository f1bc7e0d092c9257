"""Decode-batch path (moep_decode_fp64): exact fp64 ids / logits / counters for
a few tokens per step, against the oracle (predictor.py:193-240, 337-351;
metrics.py:138-193). Also the tensor-core path forced at the same tiny sizes."""
import numpy as np
import pytest
import torch

from test_gpu_parity import O, bf16_model, oracle_params, pb  # noqa: F401  (fixtures)

pytestmark = pytest.mark.gpu

SHAPES = [
    # arch, d, h, E, k
    ("arch2", 2048, 2048, 64, 6),    # DSV2L
    ("arch2", 2048, 2048, 128, 8),   # Qwen3
    ("arch2", 4096, 2048, 16, 2),    # Phi
    ("arch1", 2048, 2048, 64, 6),
    ("arch2", 100, 40, 8, 2),        # ragged d / h (not multiples of 8 / 16)
]


@pytest.mark.parametrize("arch,d,h,e,k", SHAPES)
@pytest.mark.parametrize("n", [1, 5, 8, 9, 33, 64])
def test_decode_matches_oracle(pb, O, arch, d, h, e, k, n):
    rng = np.random.default_rng(n * 131 + e)
    m = bf16_model(pb, O, arch, d, h, e, seed=7, rng=rng)
    x = O.round_bf16(rng.standard_normal((n, d)))
    zref = O.predict_logits(oracle_params(m), x)
    dev = m.to_device()
    assert n <= dev.decode_max_tokens
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    z = dev.logits(xt, validate=False).cpu().numpy()
    assert np.allclose(z, zref, rtol=0, atol=1e-11), np.abs(z - zref).max()
    for mm in sorted({1, k, min(k + 4, e), e}):
        assert np.array_equal(dev.topk(xt, mm, validate=False).cpu().numpy(), O.top_k_batch(zref, mm)), mm
    truth = O.top_k_batch(zref + 0.05 * rng.standard_normal(zref.shape), k)
    ms = O.default_m_list(k, e)
    cnt, _, ids = dev.evaluate(xt, torch.from_numpy(truth), k, ms, ids_m=k)
    c = pb.EvalCounters.from_array(cnt.cpu().numpy(), k, e, sorted(set(ms) | {k}))
    oc = O.eval_counters(zref, truth, e, ms)
    assert c.n == n and c.top1 == oc["top1_count"]
    assert c.overprov == oc["overprov_count"] and c.recall == oc["recall_count"]
    assert np.array_equal(c.per_expert_hits, oc["per_expert_hits"])
    assert np.array_equal(c.per_expert_truth, oc["per_expert_truth"])
    assert np.array_equal(ids.cpu().numpy(), O.top_k_batch(zref, k))


def test_decode_fp64_inputs_and_weights(pb, O):
    """Non-bf16 weights and fp64 / fp32 activations stay exact on the decode path."""
    rng = np.random.default_rng(4)
    m = pb.init_model("arch2", 256, 96, 16, seed=4)
    x = rng.standard_normal((13, 256))
    zref = O.predict_logits(oracle_params(m), x)
    dev = m.to_device()
    for xt in (torch.from_numpy(x).cuda(), torch.from_numpy(x).cuda().float()):
        ref = zref if xt.dtype == torch.float64 else O.predict_logits(oracle_params(m), x.astype(np.float32))
        z = dev.logits(xt).cpu().numpy()
        assert np.allclose(z, ref, rtol=0, atol=1e-12)
        assert np.array_equal(dev.topk(xt, 3).cpu().numpy(), O.top_k_batch(ref, 3))


def test_decode_ties_lower_index(pb, O):
    m = bf16_model(pb, O, "arch2", 256, 256, 16, seed=9)
    m.w2[5] = m.w2[2]
    m.w2[9] = m.w2[2]
    x = O.round_bf16(np.random.default_rng(3).standard_normal((16, 256)))
    zref = O.predict_logits(oracle_params(m), x)
    for mm in (1, 2, 3, 4):
        assert np.array_equal(pb.predict_topk_batch(m, x, mm), O.top_k_batch(zref, mm))


def test_decode_nonfinite_raises(pb, O):
    m = bf16_model(pb, O, "arch2", 64, 128, 16, seed=1)
    x = np.zeros((4, 64))
    x[1, 7] = np.inf
    with pytest.raises(pb.ConfigurationError):
        pb.predict_topk_batch(m, x, 2)


@pytest.mark.parametrize("n", [1, 3, 64])
def test_tensor_core_path_forced_small_batches(pb, O, n):
    """K1 + fix-up on decode-sized batches (decode path disabled)."""
    rng = np.random.default_rng(n)
    m = bf16_model(pb, O, "arch2", 2048, 2048, 128, seed=2, rng=rng)
    x = O.round_bf16(rng.standard_normal((n, 2048)))
    zref = O.predict_logits(oracle_params(m), x)
    dev = m.to_device()
    dev.decode_max_tokens = 0
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    assert np.array_equal(dev.topk(xt, 8).cpu().numpy(), O.top_k_batch(zref, 8))


@pytest.mark.parametrize("n", [12, 40])
def test_decode_zero_and_subnormal_bf16_operands(pb, O, n):
    """The DMMA operand conversion (bits into the fp64 hi word, one exact DMUL by
    2^896) keeps bf16 zeros and subnormals exact: rows made only of subnormals
    give logits of order 1e-39 whose ranking a flush-to-zero would lose."""
    rng = np.random.default_rng(n)
    d, h, e, k = 2048, 2048, 64, 6
    m = bf16_model(pb, O, "arch2", d, h, e, seed=3, rng=rng)
    w1 = m.w1.copy()
    w1[:, ::7] = 0.0                                   # exact zeros in W1
    w1[::5, 3::11] = rng.integers(1, 128, w1[::5, 3::11].shape) * 2.0 ** -133  # W1 subnormals
    m.w1 = w1
    x = O.round_bf16(rng.standard_normal((n, d)))
    sub = rng.integers(1, 128, (4, d)) * 2.0 ** -133 * rng.choice([-1.0, 1.0], (4, d))
    x[:4] = sub                                        # rows of bf16 subnormals only
    x[4:8, ::3] = 0.0                                  # zeros mixed into normal rows
    x[8, :] = 0.0                                      # an all-zero row
    assert np.array_equal(O.round_bf16(x), x)
    zref = O.predict_logits(oracle_params(m), x)
    assert np.abs(zref[:4]).max() < 1e-30 and np.abs(zref[:4]).max() > 0
    dev = m.to_device()
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    assert np.array_equal(xt.cpu().double().numpy(), x)
    z = dev.logits(xt, validate=False).cpu().numpy()
    assert np.allclose(z[:4], zref[:4], rtol=1e-9, atol=0), np.abs(z[:4] - zref[:4]).max()
    assert np.allclose(z, zref, rtol=0, atol=1e-11), np.abs(z - zref).max()
    assert np.array_equal(dev.topk(xt, k, validate=False).cpu().numpy(), O.top_k_batch(zref, k))
