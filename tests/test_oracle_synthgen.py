"""Pin the synthgen oracle (oracle/synthgen.py) — CPU only.

(a) against numpy itself: Philox4x64-10 raw words, standard normals from many
    keys (fast path, wedge and tail draws), pairwise summation order;
(b) against the real reference's generate_dataset (tests/golden/synthgen.npz,
    written by tests/golden/make_golden.py);
(c) the ziggurat tables compiled into the library
    (paper_2511_10676_b200/csrc/ziggurat_tables.inc) equal the oracle's own
    extraction from numpy.
"""

import os
import re

import numpy as np
import pytest

from oracle import synthgen as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ["dsv2l_identity", "nonlinear_noise", "linear_raw", "identity_noise_raw"]
# name -> (d, E, k, n, seed, transform, post_norm, sigma, nonlinear_hidden); tests/golden/make_golden.py
SPECS = {
    "dsv2l_identity": (2048, 64, 6, 24, 3, "identity", True, 0.0, 64),
    "nonlinear_noise": (256, 16, 2, 40, 5, "nonlinear", True, 0.1, 32),
    "linear_raw": (128, 128, 8, 24, 7, "linear", False, 0.0, 64),
    "identity_noise_raw": (96, 8, 3, 30, 11, "identity", False, 0.25, 64),
}


def teacher_mats(seed, d, transform, nh):
    """synthgen.py:79-90 (one numpy stream per teacher matrix set)."""
    mk = lambda idx: np.random.Generator(np.random.Philox(key=S.stream_key(seed, idx)))
    if transform == "linear":
        return {"mix": mk(S.TEACHER_KEY_OFFSET).standard_normal((d, d)) / np.sqrt(d)}
    if transform == "nonlinear":
        g = mk(S.TEACHER_KEY_OFFSET + 1)
        w_in = g.standard_normal((nh, d)) / np.sqrt(d)
        w_out = g.standard_normal((d, nh)) / np.sqrt(nh)
        return {"w_in": w_in, "w_out": w_out}
    return {}


def test_philox_raw_words_match_numpy():
    for seed, idx in [(0, 0), (7, 12345), (2**63 + 5, 2**40 + 3)]:
        key = S.stream_key(seed, idx)
        want = np.random.Philox(key=key).random_raw(40)
        s = S.PhiloxStream(key)
        assert [s.next64() for _ in range(40)] == [int(v) for v in want]


def test_standard_normal_matches_numpy():
    n_tail = 0
    for idx in range(12):
        key = S.stream_key(5, idx)
        want = np.random.Generator(np.random.Philox(key=key)).standard_normal(6000)
        s = S.PhiloxStream(key)
        got = np.array([S.standard_normal(s) for _ in range(6000)])
        assert np.array_equal(got, want)
        n_tail += int(np.sum(np.abs(want) > S.ZIG_R))
    assert n_tail > 0  # the tail branch was exercised


def test_pairwise_sum_matches_numpy_reductions():
    rng = np.random.default_rng(3)
    for d in (2048, 2047, 1000, 130, 129, 128, 64, 9, 7, 2):
        x = rng.standard_normal((8, d)) * np.exp(3 * rng.standard_normal((8, d)))
        for i in range(8):
            s = S.pairwise_sum(x[i])
            assert s == x[i].sum()
            m = s / d
            assert m == x[i].mean()
            assert S.pairwise_sum((x[i] - m) * (x[i] - m)) / d == x[i].var()


def test_compiled_tables_equal_oracle_extraction():
    ki, wi, fi = S.extract_tables()
    src = open(os.path.join(ROOT, "paper_2511_10676_b200", "csrc", "ziggurat_tables.inc")).read()

    def block(name):
        body = src[src.index(name):]
        body = body[body.index("{") + 1:body.index("};")]
        return [t.strip() for t in body.replace("\n", " ").split(",") if t.strip()]

    k_c = [int(t.rstrip("ul"), 16) for t in block("kZigKi")]
    w_c = [float.fromhex(t) for t in block("kZigWi")]
    f_c = [float.fromhex(t) for t in block("kZigFi")]
    assert k_c == [int(v) for v in ki]
    assert w_c == [float(v) for v in wi]
    assert f_c == [float(v) for v in fi]


@pytest.mark.parametrize("case", CASES)
def test_oracle_generate_dataset_matches_reference(golden, case):
    g = golden("synthgen")
    d, e, k, n, seed, transform, post_norm, sigma, nh = SPECS[case]
    mats = teacher_mats(seed, d, transform, nh)
    x32, s32, topk, _ = S.generate_dataset(g[case + "_gate"], k, n, seed=seed, transform=transform,
                                           post_norm=post_norm, noise_sigma=sigma, **mats)
    assert np.array_equal(x32, g[case + "_x"])
    assert np.array_equal(s32, g[case + "_scores"])
    assert np.array_equal(topk, g[case + "_topk"])
    # raw per-sample streams (activation row then noise row)
    for i in range(2):
        x, nz = S.sample_normals(seed, i, d, True)
        assert np.array_equal(np.concatenate([x, nz]), g[case + "_raw"][i])


def test_layer_norm_golden(golden):
    g = golden("synthgen")
    for d in (2048, 1000, 129, 7):
        assert np.array_equal(S.layer_norm(g[f"ln_{d}_x"]), g[f"ln_{d}_y"])
