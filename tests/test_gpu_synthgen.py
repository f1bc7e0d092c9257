"""K11 synthetic teacher on the GPU (paper_2511_10676_b200.synthgen) against
the real reference's generate_dataset (tests/golden/synthgen.npz) and the
oracle (oracle/synthgen.py).

Tolerances (csrc/synthgen.cu header): Philox words, the ziggurat fast path and
the pairwise sums are exact, so activations (float32) and layer-norm outputs
must be bit-identical; CUDA exp / log1p may differ from glibc by one ulp, so
fp64 normals may differ by one ulp only on tail draws (|x| > 3.654); the gate
GEMM runs on cuBLAS instead of OpenBLAS, so float32 scores may differ by one
float32 ulp and top-k ids must match wherever the scores do.
"""
import numpy as np
import pytest
import torch

from test_oracle_synthgen import CASES, SPECS, teacher_mats

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_10676_b200 import synthgen
    return synthgen


@pytest.fixture(scope="module")
def S():
    from oracle import synthgen
    return synthgen


def teacher(sg, g, case):
    d, e, k, n, seed, transform, post_norm, sigma, nh = SPECS[case]
    router = sg.RouterSpec(d, e, k, g[case + "_gate"])
    return sg.TeacherSpec(router, transform=transform, post_norm=post_norm, noise_sigma=sigma,
                          nonlinear_hidden=nh, seed=seed), n


def check_scores(s_gpu, s_ref, t_gpu, t_ref):
    np.testing.assert_array_max_ulp(s_gpu, s_ref, maxulp=1)
    same = np.all(s_gpu == s_ref, axis=1)
    assert same.mean() >= 0.9
    assert np.array_equal(t_gpu[same], t_ref[same])


@pytest.mark.parametrize("case", CASES)
def test_generate_dataset_matches_reference(sg, golden, case):
    g = golden("synthgen")
    t, n = teacher(sg, g, case)
    data = sg.generate_dataset(t, n)
    assert data.activations.dtype == np.float32 and data.true_topk.dtype == np.int64
    assert np.array_equal(data.activations, g[case + "_x"])
    check_scores(data.true_scores, g[case + "_scores"], data.true_topk, g[case + "_topk"])


def test_raw_normals_match_reference_streams(sg, golden, S):
    from paper_2511_10676_b200._lib import check, lib, ptr
    g = golden("synthgen")
    for case in CASES:
        d, seed = SPECS[case][0], SPECS[case][4]
        x = torch.empty((2, d), dtype=torch.float64, device="cuda")
        nz = torch.empty((2, d), dtype=torch.float64, device="cuda")
        check(lib().moep_teacher_normals(seed, 0, 2, d, 1, ptr(x), None, ptr(nz),
                                         torch.cuda.current_stream().cuda_stream), "normals")
        got = torch.cat([x, nz], dim=1).cpu().numpy()
        want = g[case + "_raw"]
        diff = got != want
        # only tail draws may differ, by at most one ulp
        assert np.all(np.abs(want[diff]) > S.ZIG_R)
        np.testing.assert_array_max_ulp(got, want, maxulp=1)


def test_many_samples_chunked_vs_oracle(sg, S):
    """4000 DSV2L-shaped samples in uneven chunks (first_index offsets across
    kernel launches); a spread of rows checked against the oracle's streams."""
    d, e, k = 2048, 64, 6
    gate = np.random.default_rng(1).standard_normal((e, d)) / np.sqrt(d)
    t = sg.TeacherSpec(sg.RouterSpec(d, e, k, gate), noise_sigma=0.05, seed=42)
    dt = sg.generate_dataset_device(t, 4000, chunk_rows=1500)
    acts = dt.activations.cpu().numpy()
    rows = [0, 1, 127, 128, 1499, 1500, 1501, 2999, 3000, 3999]
    for r in rows:
        x_o, s_o, t_o, _ = S.generate_dataset(gate, k, 1, seed=42, noise_sigma=0.05, first_index=r)
        assert np.array_equal(acts[r], x_o[0]), r
        check_scores(dt.true_scores[r:r + 1].cpu().numpy(), s_o, dt.true_topk[r:r + 1].cpu().numpy().astype(np.int64),
                     t_o)
    # every stored label set is the top-k of the stored float32 scores
    s = dt.true_scores.cpu().numpy().astype(np.float64)
    want = np.sort(np.argsort(-s, axis=1, kind="stable")[:, :k], axis=1)
    assert np.array_equal(dt.true_topk.cpu().numpy(), want)


def test_layer_norm_bit_identical_to_numpy(golden):
    import paper_2511_10676_b200 as pb
    g = golden("synthgen")
    for d in (2048, 1000, 129, 7):
        assert np.array_equal(pb.layer_norm(g[f"ln_{d}_x"]), g[f"ln_{d}_y"])
    x = np.random.default_rng(0).standard_normal((3, 5, 300)) * 10
    from oracle import synthgen as S
    assert np.array_equal(pb.layer_norm(x), S.layer_norm(x))


def test_teacher_errors(sg):
    from paper_2511_10676_b200.exceptions import ConfigurationError
    r = sg.RouterSpec(16, 4, 2, np.ones((4, 16)))
    with pytest.raises(ConfigurationError):
        sg.TeacherSpec(r, transform="cubic")
    with pytest.raises(ConfigurationError):
        sg.TeacherSpec(r, noise_sigma=-1.0)
    with pytest.raises(ConfigurationError):
        sg.RouterSpec(16, 4, 5, np.ones((4, 16)))
    with pytest.raises(ValueError):
        sg.generate_dataset(sg.TeacherSpec(r), 0)


def test_softmax_numpy_order():
    """core.softmax (core.py:19-24) on the device: within an ulp of numpy (CUDA
    exp vs numpy's SIMD exp), any axis, and ranking-preserving like the
    reference's test (test_core.py:134-147)."""
    import paper_2511_10676_b200 as pb
    from oracle import synthgen as S
    rng = np.random.default_rng(5)
    for shape, axis in [((1000, 64), -1), ((300, 128), 0), ((4, 7, 33), 1), ((2, 5000), -1)]:
        z = rng.standard_normal(shape) * 4
        got = pb.softmax(z, axis=axis)
        want = np.moveaxis(S.softmax(np.moveaxis(z, axis, -1)), -1, axis)
        np.testing.assert_allclose(got, want, rtol=4e-16 * 8, atol=0)
    z = rng.standard_normal((1000, 64))
    assert np.array_equal(np.argsort(-pb.softmax(z), axis=1, kind="stable"), np.argsort(-z, axis=1, kind="stable"))


@pytest.mark.parametrize("M,N,K,epi", [(1000, 64, 2048, 0), (333, 130, 77, 1), (4096, 2048, 512, 0), (7, 5, 3, 1)])
def test_dgemm_nt_vs_numpy(M, N, K, epi):
    """moep_dgemm_nt (the teacher's GEMMs on the fp64 tensor cores) against
    numpy float64, ragged shapes and the tanh epilogue."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_10676_b200._lib import check, lib, ptr
    rng = np.random.default_rng(M + N + K)
    a = rng.standard_normal((M, K))
    b = rng.standard_normal((N, K)) / np.sqrt(K)
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c = torch.empty((M, N), dtype=torch.float64, device="cuda")
    check(lib().moep_dgemm_nt(ptr(at), K, ptr(bt), K, ptr(c), N, M, N, K, epi,
                              torch.cuda.current_stream().cuda_stream), "moep_dgemm_nt")
    ref = a @ b.T
    if epi:
        ref = np.tanh(ref)
    assert np.allclose(c.cpu().numpy(), ref, rtol=1e-12, atol=1e-13)
