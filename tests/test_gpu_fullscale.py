"""Full-scale parity (SURVEY §7 hard part 6): one whole C2 layer (1,048,576
tokens, DSV2L shape) and the C3 Qwen3 shape over 48 layers x 65,536 tokens,
both on the oracle-gate workload (workloads.py: the true experts sit at the k
boundary, so the near-tie fix-up is exercised at a realistic rate).

The checker at these sizes is the exact fp64 path on the GPU (the fix-up's
fp64 DMMA GEMM over every row), itself pinned to the CPU oracle here on a
sample and in test_gpu_parity.py; counters are rebuilt from the fp64 logits
by K7. Bit-exact ids and counters are required on every token."""

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


def _check_layer(pb, O, model, x, truth, k, ms, n_oracle):
    from paper_2511_10676_b200.engine import eval_logits_device, topk_logits_device
    dev = model.to_device()
    e = model.n_experts
    cnt, fcount, ids = dev.evaluate(x, truth, k, ms, ids_m=k)
    z64 = dev.fp64_rows(x, torch.empty((x.shape[0], e), dtype=torch.float64, device="cuda"))
    ids64 = topk_logits_device(z64, k)
    bad = int((ids64 != ids).any(dim=1).sum())
    c64 = eval_logits_device(z64, truth, k, e, ms)
    # K1's raw error on this layer, against the margin contract
    lg = torch.empty((x.shape[0], e), dtype=torch.float32, device="cuda")
    dev._k1(x, logits=lg)
    w1 = torch.as_tensor(model.w1, dtype=torch.float32, device="cuda")
    a = x.float() @ w1.T
    hn = torch.linalg.vector_norm(a * torch.sigmoid(a), dim=1).double()
    ratio = float(((lg.double() - z64).abs().amax(1) / (hn * dev.w2_norm)).max())
    # the CPU oracle on a sample
    rows = np.linspace(0, x.shape[0] - 1, n_oracle).astype(np.int64)
    p = {"arch": "arch2", "w1": model.w1, "b1": model.b1, "w2": model.w2, "b2": model.b2}
    zo = O.predict_logits(p, x[rows].double().cpu().numpy())
    assert np.allclose(z64[rows].cpu().numpy(), zo, rtol=0, atol=1e-11)
    assert np.array_equal(ids[rows].cpu().numpy(), O.top_k_batch(zo, k))
    return bad, bool(torch.equal(cnt, c64)), int(fcount.item()), ratio, dev.tau_rel


def test_full_c2_layer_bit_exact(pb):
    import workloads as W
    from oracle import oracle as O
    n = 1 << 20
    model, x, truth = W.make_layer("gate", 2048, 2048, 64, 6, n, seed=77, device="cuda")
    bad, same, nflag, ratio, tau = _check_layer(pb, O, model, x, truth, 6, [6, 10, 64], 2048)
    assert bad == 0
    assert same
    assert 0 < nflag < n // 50
    assert 4 * ratio <= tau, ratio


def test_qwen3_48_layers_bit_exact(pb):
    import workloads as W
    from oracle import oracle as O
    n = 1 << 16
    worst = 0.0
    for layer in range(48):
        model, x, truth = W.make_layer("gate", 2048, 2048, 128, 8, n, seed=500 + layer, device="cuda")
        bad, same, _, ratio, tau = _check_layer(pb, O, model, x, truth, 8, [8, 12, 128], 64)
        assert bad == 0, layer
        assert same, layer
        worst = max(worst, ratio)
    # v4 at E = 128 keeps one z accumulator: its margin is 1.5 tau (k1v4_predict.cu)
    assert 4 * worst <= 1.5 * tau, worst
