"""The drop-in boundary, exercised on the real reference: the unmodified
`moepredict` package (installed into baseline/_ref by `pip install --target`,
DESIGN §8) is run once as shipped and once after patch_reference(); results
must agree (ids, counters and EvalResult fields exactly; fp64 logits, losses
and trained parameters to fp64 round-off). Also our own ExpertPredictor's
sklearn contract (reference tests/test_estimator.py:27-45) and the
DevicePredictor cache of the numpy API."""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.isdir(os.path.join(REF, "moepredict")):
        pytest.skip("baseline/_ref/moepredict is not installed (see DESIGN §8)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import moepredict
    return moepredict


@pytest.fixture
def patched(ref):
    from paper_2511_10676_b200.integration import patch_reference, unpatch_reference
    names = patch_reference("moepredict")
    yield names
    unpatch_reference()


def _bf16(a):
    a = np.asarray(a, dtype=np.float64)
    m, e = np.frexp(a)
    return np.ldexp(np.rint(m * 256.0), e - 8)


def test_patch_rebinds_import_time_names(ref, patched):
    import moepredict.estimator as E
    import moepredict.metrics as M
    import moepredict.trainer as T
    from paper_2511_10676_b200 import integration  # noqa: F401
    for name in ("moepredict.metrics.predict_logits", "moepredict.trainer.forward", "moepredict.trainer.backward",
                 "moepredict.trainer.loss_and_grad", "moepredict.trainer.evaluate_predictions",
                 "moepredict.estimator.train", "moepredict.estimator.predict_topk_batch",
                 "moepredict.estimator.evaluate_predictions", "moepredict.evaluate", "moepredict.train",
                 "moepredict.forward", "moepredict.predict_topk", "moepredict.loss_and_grad"):
        assert name in patched, name
    assert M.predict_logits.__module__.startswith("paper_2511_10676_b200")
    assert T.train is not None and E.train.__wrapped__.__module__.startswith("paper_2511_10676_b200")


def test_predictor_calls_match_unpatched(ref):
    from moepredict import predictor as P
    from paper_2511_10676_b200.integration import patch_reference, unpatch_reference
    rng = np.random.default_rng(0)
    m = P.init_model("arch2", 2048, 2048, 64, seed=0)
    m.w1, m.w2 = _bf16(m.w1), _bf16(m.w2)
    x = _bf16(rng.standard_normal((4096, 2048)))
    ids_ref = P.predict_topk_batch(m, x[:1024], 6)
    z_ref = P.predict_logits(m, x[:1024])
    sel_ref = P.predict_topk(m, x[5], 10)
    patch_reference()
    try:
        ids = P.predict_topk_batch(m, x[:1024], 6)
        z = P.predict_logits(m, x[:1024])
        sel = P.predict_topk(m, x[5], 10)
        assert isinstance(sel, type(sel_ref))
        assert np.array_equal(ids, ids_ref) and ids.dtype == ids_ref.dtype
        assert np.allclose(z, z_ref, rtol=0, atol=1e-11)
        assert np.array_equal(sel.indices, sel_ref.indices)
        # the reference's exception classes cross the boundary
        bad = x[:4].copy()
        bad[1, 2] = np.inf
        from moepredict.exceptions import ConfigurationError
        with pytest.raises(ConfigurationError):
            P.predict_logits(m, bad)
        with pytest.raises(ValueError):
            P.predict_topk_batch(m, x[:4], 65)
    finally:
        unpatch_reference()


def test_evaluate_and_losses_match_unpatched(ref):
    import moepredict
    from moepredict.core import RouterSpec
    from moepredict.losses import BatchLabels, LossSpec
    from moepredict.synthgen import TeacherSpec, generate_dataset
    from paper_2511_10676_b200.integration import patch_reference, unpatch_reference
    rng = np.random.default_rng(3)
    router = RouterSpec(64, 16, 2, rng.standard_normal((16, 64)) / 8.0)
    data = generate_dataset(TeacherSpec(router=router, seed=2), 3000)
    m = moepredict.init_model("arch2", 64, 128, 16, seed=1)
    r0 = moepredict.evaluate(m, data)
    labels = BatchLabels.from_scores(data.true_scores[:256].astype(np.float64), 2)
    z = moepredict.predictor.predict_logits(m, data.activations[:256].astype(np.float64))
    losses0 = {f: moepredict.loss_and_grad(LossSpec(f), z, labels) for f in ("mse", "wbce", "focal", "ranking")}
    patch_reference()
    try:
        r1 = moepredict.evaluate(m, data)
        assert type(r1) is type(r0)
        for f in ("exact_match", "top1", "overprov", "overprov_recall", "n_samples"):
            assert getattr(r1, f) == getattr(r0, f), f
        assert np.array_equal(r1.per_expert_hits, r0.per_expert_hits)
        assert np.array_equal(r1.per_expert_truth, r0.per_expert_truth)
        assert np.allclose(r1.tier_profile, r0.tier_profile, rtol=1e-12, atol=0)
        data2 = moepredict.generate_dataset(TeacherSpec(router=router, seed=2), 3000)
        assert np.array_equal(data2.true_topk, data.true_topk)
        for f, (l0, g0) in losses0.items():
            l1, g1 = moepredict.loss_and_grad(LossSpec(f), z, labels)
            assert abs(l1 - l0) <= 1e-12 * max(1.0, abs(l0)), f
            assert np.allclose(g1, g0, rtol=1e-10, atol=1e-14), f
        with pytest.raises(IndexError):
            moepredict.metrics.evaluate_predictions(z, np.full((256, 2), 16), 16)
    finally:
        unpatch_reference()


def test_train_matches_unpatched(ref):
    import moepredict
    from moepredict.core import RouterSpec
    from moepredict.losses import LossSpec
    from moepredict.synthgen import TeacherSpec, generate_dataset
    from moepredict.trainer import TrainConfig
    from paper_2511_10676_b200.integration import patch_reference, unpatch_reference
    rng = np.random.default_rng(5)
    router = RouterSpec(32, 8, 2, rng.standard_normal((8, 32)) / 4.0)
    data = generate_dataset(TeacherSpec(router=router, seed=7), 1200)
    cfg = TrainConfig(loss=LossSpec("ranking"), hidden=48, epochs=2, batch_size=128, seed=3)
    m0, rep0 = moepredict.train(cfg, data)
    patch_reference()
    try:
        m1, rep1 = moepredict.train(cfg, data)
        assert type(m1) is type(m0) and type(rep1) is type(rep0)
        for name in ("w1", "b1", "w2", "b2"):
            assert np.allclose(getattr(m1, name), getattr(m0, name), rtol=1e-8, atol=1e-10), name
        for e0, e1 in zip(rep0.epochs, rep1.epochs):
            assert e1.train_loss == pytest.approx(e0.train_loss, rel=1e-9)
            assert (e0.exact_match, e0.top1, e0.overprov) == (e1.exact_match, e1.top1, e1.overprov)
    finally:
        unpatch_reference()


def test_estimator_fit_predict_score_clone_match_unpatched(ref):
    from moepredict.core import RouterSpec
    from moepredict.estimator import ExpertPredictor
    from moepredict.synthgen import TeacherSpec, generate_dataset
    from sklearn.base import clone
    from paper_2511_10676_b200.integration import patch_reference, unpatch_reference
    rng = np.random.default_rng(11)
    router = RouterSpec(12, 6, 2, rng.standard_normal((6, 12)) / 3.0)
    data = generate_dataset(TeacherSpec(router=router, seed=4), 1500)
    X, y = data.activations.astype(np.float64), data.true_scores.astype(np.float64)
    est0 = ExpertPredictor(k=2, hidden=48, epochs=3, random_state=3).fit(X[:1200], y[:1200])
    p0, s0, d0 = est0.predict(X[1200:]), est0.score(X[1200:], y[1200:]), est0.decision_function(X[1200:])
    patch_reference()
    try:
        est1 = ExpertPredictor(k=2, hidden=48, epochs=3, random_state=3).fit(X[:1200], y[:1200])
        assert np.array_equal(est1.predict(X[1200:]), p0)
        assert est1.score(X[1200:], y[1200:]) == s0
        assert np.allclose(est1.decision_function(X[1200:]), d0, rtol=1e-8, atol=1e-10)
        fresh = clone(est1)
        assert fresh.get_params() == est1.get_params() and not hasattr(fresh, "model_")
    finally:
        unpatch_reference()


def test_own_estimator_sklearn_contract():
    """Our ExpertPredictor keeps the reference's get_params / clone contract
    (tests/test_estimator.py:27-45) and fits / predicts on the device."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from sklearn.base import clone
    from sklearn.exceptions import NotFittedError
    import paper_2511_10676_b200 as pb
    from paper_2511_10676_b200 import synthgen as sg
    est = pb.ExpertPredictor(hidden=99, loss="ranking")
    params = est.get_params()
    assert params["hidden"] == 99
    assert pb.ExpertPredictor().set_params(**params).get_params() == params
    with pytest.raises(NotFittedError):
        pb.ExpertPredictor().predict(np.zeros((2, 4)))
    rng = np.random.default_rng(11)
    t = sg.TeacherSpec(sg.RouterSpec(12, 6, 2, rng.standard_normal((6, 12)) / 3.0), seed=4)
    data = sg.generate_dataset(t, 1500)
    X, y = data.activations.astype(np.float64), data.true_scores.astype(np.float64)
    fitted = pb.ExpertPredictor(k=2, hidden=48, epochs=4, random_state=3).fit(X[:1200], y[:1200])
    pred = fitted.predict(X[1200:])
    assert pred.shape == (300, 2) and (pred[:, 0] < pred[:, 1]).all()
    assert fitted.decision_function(X[1200:]).shape == (300, 6)
    assert fitted.predict_topk(X[1200:], 3).shape == (300, 3)
    assert 0.0 <= fitted.score(X[1200:], y[1200:]) <= 1.0
    fresh = clone(fitted)
    assert fresh.get_params() == fitted.get_params() and not hasattr(fresh, "model_")


def test_numpy_api_reuses_the_device_copy():
    """predict_logits / predict_topk_batch on a host model upload it once; an
    in-place update (what an optimizer does) or a new array re-uploads."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2511_10676_b200 as pb
    from paper_2511_10676_b200.predictor import device_for
    rng = np.random.default_rng(1)
    m = pb.init_model("arch2", 256, 256, 16, seed=1)
    x = _bf16(rng.standard_normal((600, 256)))
    a = device_for(m)
    pb.predict_topk_batch(m, x, 2)
    assert device_for(m) is a
    z0 = pb.predict_logits(m, x)
    m.w1 -= 1e-3 * np.sign(m.w1)          # in place, every element
    b = device_for(m)
    assert b is not a
    assert not np.allclose(pb.predict_logits(m, x), z0)
    m.w2 = m.w2.copy()                    # a new array
    assert device_for(m) is not b


def test_own_public_api_vs_reference(ref):
    """Our evaluate_predictions / evaluate / compare_losses (metrics.py:138-207,
    trainer.py:207-230) against the unmodified reference on the same data."""
    import moepredict
    from moepredict.core import RouterSpec
    from moepredict.synthgen import TeacherSpec, generate_dataset
    import paper_2511_10676_b200 as pb
    rng = np.random.default_rng(9)
    router = RouterSpec(24, 8, 2, rng.standard_normal((8, 24)) / 5.0)
    data = generate_dataset(TeacherSpec(router=router, seed=1), 900)
    ours_data = pb.TraceFile(data.hidden_dim, data.n_experts, data.k, data.activations, data.true_scores,
                             data.true_topk)
    m = moepredict.init_model("arch2", 24, 40, 8, seed=2)
    z = moepredict.predictor.predict_logits(m, data.activations.astype(np.float64))
    for m_list in (None, [2, 3, 8], [4]):
        r0 = moepredict.metrics.evaluate_predictions(z, data.true_topk, 8, m_list, data.true_scores)
        r1 = pb.evaluate_predictions(z, data.true_topk, 8, m_list, data.true_scores)
        for f in ("exact_match", "top1", "overprov", "overprov_recall", "n_samples", "k", "n_experts"):
            assert getattr(r1, f) == getattr(r0, f), (f, m_list)
        assert np.array_equal(r1.per_expert_hits, r0.per_expert_hits)
        assert np.allclose(r1.tier_profile, r0.tier_profile, rtol=1e-12, atol=0)
    with pytest.raises(ValueError):
        pb.evaluate_predictions(z, data.true_topk, 8, [1])
    with pytest.raises(IndexError):
        pb.evaluate_predictions(z, np.full_like(data.true_topk, 8), 8)
    with pytest.raises(ValueError):
        pb.evaluate_predictions(z, np.full_like(data.true_topk, -1), 8)
    # a repeated true id counts twice, as the reference's bincount does
    dup = data.true_topk.copy()
    dup[:, 1] = dup[:, 0]
    r0 = moepredict.metrics.evaluate_predictions(z, dup, 8)
    r1 = pb.evaluate_predictions(z, dup, 8)
    assert np.array_equal(r1.per_expert_hits, r0.per_expert_hits)
    assert np.array_equal(r1.per_expert_truth, r0.per_expert_truth)
    assert (r1.exact_match, r1.top1, r1.overprov) == (r0.exact_match, r0.top1, r0.overprov)
    e0 = moepredict.evaluate(m, data)
    e1 = pb.evaluate(pb.PredictorModel("arch2", m.w1, m.b1, m.w2, m.b2), ours_data)
    assert (e1.exact_match, e1.top1, e1.overprov, e1.overprov_recall) == \
        (e0.exact_match, e0.top1, e0.overprov, e0.overprov_recall)
    from moepredict.trainer import TrainConfig, compare_losses
    cfg = TrainConfig(hidden=16, batch_size=128, seed=4)
    rows0 = compare_losses(cfg, data)
    rows1 = pb.compare_losses(pb.TrainConfig(hidden=16, batch_size=128, seed=4), ours_data)
    assert len(rows0) == len(rows1) == 8
    for a, b in zip(rows0, rows1):
        assert (a["loss"], a["arch"]) == (b["loss"], b["arch"])
        for f in ("exact_match", "top1", "overprov"):
            assert a[f] == b[f], (a, b)
