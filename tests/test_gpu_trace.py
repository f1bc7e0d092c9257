"""K10 MOEPA1 ingestion on the GPU (trace_io) against files and exception kinds
produced by the real reference (tests/golden/make_golden.py): arrays
bit-identical to the reference's read_trace (synthgen.py:219-253), the same
exception class and message for every corruption, byte-identical write_trace,
multi-chunk streaming."""
import os

import numpy as np
import pytest
import torch

from trace_corrupt import corruptions

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def tio():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_10676_b200 import trace_io
    return trace_io


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(HERE, "trace.npz"))


@pytest.mark.parametrize("chunk_bytes", [64 << 20, 1000])
def test_read_matches_reference(tio, g, chunk_bytes):
    t = tio.read_trace_device(os.path.join(HERE, "trace_small.moepa"), chunk_bytes=chunk_bytes)
    assert [t.hidden_dim, t.n_experts, t.k, len(t)] == g["dims"].tolist()
    h = t.to_host()
    assert np.array_equal(h.activations, g["acts"])
    assert np.array_equal(h.true_scores, g["scores"])
    assert np.array_equal(h.true_topk, g["topk"]) and h.true_topk.dtype == np.int64


def test_bf16_activations_and_ties(tio, g):
    t = tio.read_trace_device(os.path.join(HERE, "trace_small.moepa"), act_dtype=torch.bfloat16)
    assert t.activations.dtype == torch.bfloat16
    ref = torch.from_numpy(g["acts"]).to(torch.bfloat16)
    assert torch.equal(t.activations.cpu(), ref)
    ties = tio.read_trace(os.path.join(HERE, "trace_ties.moepa"))
    assert np.array_equal(ties.true_topk, g["tie_topk"])


def test_corruptions_raise_reference_exceptions(tio, g, tmp_path):
    import paper_2511_10676_b200 as pb
    blob = open(os.path.join(HERE, "trace_small.moepa"), "rb").read()
    d, e, k, _n = g["dims"].tolist()
    bad = corruptions(blob, d, e, k)
    for name, kind, msg in zip(g["corrupt_names"], g["corrupt_kinds"], g["corrupt_msgs"]):
        p = tmp_path / f"{name}.moepa"
        p.write_bytes(bad[str(name)])
        with pytest.raises(getattr(pb, str(kind))) as ei:
            tio.read_trace_device(str(p), chunk_bytes=2000)
        assert type(ei.value).__name__ == kind and str(ei.value) == msg, name


def test_write_trace_same_bytes(tio, g, tmp_path):
    from paper_2511_10676_b200.data import TraceFile
    d, e, k, n = g["dims"].tolist()
    tf = TraceFile(d, e, k, g["acts"], g["scores"], g["topk"])
    p = tmp_path / "w.moepa"
    tio.write_trace(str(p), tf)
    assert p.read_bytes() == open(os.path.join(HERE, "trace_small.moepa"), "rb").read()
    import paper_2511_10676_b200 as pb
    with pytest.raises(pb.DataError):
        tio.write_trace(str(tmp_path / "e.moepa"), TraceFile(d, e, k, g["acts"][:0], g["scores"][:0], g["topk"][:0]))
    bad = TraceFile(d, e, k, g["acts"], g["scores"], g["topk"][:, ::-1].copy())
    with pytest.raises(pb.RecordValidationError):
        tio.write_trace(str(tmp_path / "b.moepa"), bad)


def test_large_trace_streams_in_chunks(tio, tmp_path):
    """DSV2L-shaped records (d=2048, E=64, k=6), 3000 records in ~1 MB chunks."""
    from paper_2511_10676_b200.data import make_dataset
    rng = np.random.default_rng(3)
    n, d, e, k = 3000, 2048, 64, 6
    acts = rng.standard_normal((n, d)).astype(np.float32)
    logits = rng.standard_normal((n, e))
    sc = np.exp(logits - logits.max(1, keepdims=True))
    sc /= sc.sum(1, keepdims=True)
    tf = make_dataset(acts, sc, k)
    p = tmp_path / "big.moepa"
    tio.write_trace(str(p), tf)
    t = tio.read_trace_device(str(p), chunk_bytes=1 << 20)
    assert torch.equal(t.activations.cpu(), torch.from_numpy(tf.activations))
    assert torch.equal(t.true_scores.cpu(), torch.from_numpy(tf.true_scores))
    assert np.array_equal(t.true_topk.cpu().numpy(), tf.true_topk)
