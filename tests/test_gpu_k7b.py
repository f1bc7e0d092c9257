"""K7 from given logits, one thread per token (k7b_rows.cu: packed 32-bit keys,
bitonic top-G networks, exact fallback at ambiguous boundaries) against the
oracle (numpy argsort(-z, stable) semantics: descending value, ties to the lower
index, -0.0 == +0.0, NaN last): ids and every evaluation counter bit-exact,
on adversarial rows: exact ties, keys equal in their top 26 bits, signed zeros,
infinities, NaN, ragged row counts, fp32 and fp64, thresholds beyond the list."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def O():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from oracle import oracle
    return oracle


def _rows(n, e, seed, dtype):
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((n, e))
    q = n // 6
    z[:q] = np.round(z[:q] * 2) / 2                          # heavy exact ties
    base = rng.standard_normal((q, 1))
    ulp = np.spacing(np.abs(base).astype(dtype)).astype(np.float64)
    z[q: 2 * q] = base + ulp * rng.integers(-3, 4, (q, e))   # equal in the top bits, distinct values
    z[2 * q: 2 * q + 8] = 0.0
    z[2 * q: 2 * q + 8, ::3] = -0.0                          # signed zeros
    z[2 * q + 8: 2 * q + 16, 1::5] = np.inf
    z[2 * q + 16: 2 * q + 24, 2::7] = -np.inf
    z[2 * q + 24: 2 * q + 32, ::4] = np.nan                  # NaN last in numpy's order
    return z.astype(dtype)


def _oracle_topk(z, m):
    # numpy's stable argsort of -z (NaN last), ascending ids: core.top_k_batch
    order = np.argsort(-z.astype(np.float64), axis=1, kind="stable")
    return np.sort(order[:, :m], axis=1)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("e", [16, 32, 64])
def test_k7b_topk_vs_oracle(O, dtype, e):
    from paper_2511_10676_b200.engine import topk_logits_device
    n = 4133  # ragged: not a multiple of 32 rows per warp
    z = _rows(n, e, e + (8 if dtype == np.float64 else 0), dtype)
    zt = torch.from_numpy(z).cuda()
    for m in (1, 2, 6, 7, 8, 10, 15):
        got = topk_logits_device(zt, m).cpu().numpy()
        ref = _oracle_topk(z, m)
        bad = np.nonzero((got != ref).any(axis=1))[0]
        assert bad.size == 0, (m, bad[:5], z[bad[:1]], got[bad[:1]], ref[bad[:1]])
    finite = np.isfinite(z).all(axis=1)
    assert np.array_equal(topk_logits_device(zt, 6).cpu().numpy()[finite], O.top_k_batch(z[finite], 6))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("e,k,ms", [(64, 6, [6, 10, 64]), (64, 6, [1, 6, 20, 64]), (32, 4, [4, 8, 15]),
                                    (16, 2, [2, 3, 16]), (64, 15, [15, 64])])
def test_k7b_eval_vs_oracle(O, dtype, e, k, ms):
    from paper_2511_10676_b200.engine import EvalCounters, eval_logits_device
    n = 5021
    rng = np.random.default_rng(k * 100 + e)
    z = _rows(n, e, k + e, dtype)
    z = np.where(np.isnan(z), 0.0, z).astype(dtype)  # the oracle's rank_order is numpy's; keep it NaN-free
    truth = np.stack([rng.choice(e, k, replace=False) for _ in range(n)]).astype(np.int32)
    truth[::97, 1 % k] = truth[::97, 0]  # repeated true ids count each time (bincount)
    c = eval_logits_device(torch.from_numpy(z).cuda(), torch.from_numpy(truth), k, e, ms).cpu().numpy()
    got = EvalCounters.from_array(c, k, e, ms)
    ref = O.eval_counters(z.astype(np.float64), truth, e, ms)
    assert got.n == ref["n"] and got.top1 == ref["top1_count"]
    for m in ms:
        assert got.overprov[m] == ref["overprov_count"][m], m
        assert got.recall[m] == ref["recall_count"][m], m
    assert np.array_equal(got.per_expert_hits, ref["per_expert_hits"])
    assert np.array_equal(got.per_expert_truth, ref["per_expert_truth"])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("e,k", [(16, 2), (32, 4), (64, 6)])
def test_k3_labels_rows_vs_oracle(O, dtype, e, k):
    """K3 (moep_labels) one thread per token: rank_of, topk_mask and the strict
    pairs among the top min(10, E) (losses.py:198-207) equal the oracle's on
    adversarial rows (exact ties, near-ties, signed zeros, infinities)."""
    from paper_2511_10676_b200._lib import check, lib, ptr, dtype_code
    n = 3001
    z = _rows(n, e, 7 * e + k, dtype)
    z = np.where(np.isnan(z), 0.25, z).astype(dtype)
    s = torch.from_numpy(z).cuda()
    rank = torch.empty((n, e), dtype=torch.int32, device="cuda")
    mask = torch.empty((n, e), dtype=torch.uint8, device="cuda")
    pairs = torch.empty(n, dtype=torch.int32, device="cuda")
    check(lib().moep_labels(ptr(s), dtype_code(s), n, e, k, ptr(rank), ptr(mask), ptr(pairs), None), "moep_labels")
    ref = O.batch_labels(z.astype(np.float64), k)
    assert np.array_equal(rank.cpu().numpy(), ref["rank_of"])
    assert np.array_equal(mask.cpu().numpy().astype(bool), ref["topk_mask"])
    top_cut = min(10, e)
    zz = z.astype(np.float64)
    want = np.array([int(((zz[i][ref["rank_of"][i] <= top_cut])[:, None] >
                          (zz[i][ref["rank_of"][i] <= top_cut])[None, :]).sum()) for i in range(n)])
    assert np.array_equal(pairs.cpu().numpy(), want)
