"""GPU tests of the prefetch path: K8 plan == numpy union minus resident,
copy-engine and SM-gather (K9) loads land the right bytes in the right slots."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_10676_b200 import prefetch
    return prefetch


def test_plan_union_minus_resident(pf):
    rng = np.random.default_rng(0)
    E, eb = 64, 4096
    store = pf.ExpertStore(E, eb)
    cache = pf.ExpertCache(32, eb, E)
    p = pf.Prefetcher(store, cache)
    for trial in range(20):
        B = int(rng.integers(1, 40))
        ids = np.sort(rng.permuted(np.tile(np.arange(E), (B, 1)), axis=1)[:, :6], axis=1)
        resident = rng.choice(E, size=int(rng.integers(0, 10)), replace=False)
        cache.reset()
        if len(resident):
            cache.slot_of[torch.as_tensor(resident).cuda().long()] = 0
        p.plan(torch.as_tensor(ids).cuda())
        torch.cuda.synchronize()
        n = int(p.need_count.item())
        want = sorted(set(ids.ravel().tolist()) - set(resident.tolist()))
        assert p.need_list[:n].cpu().tolist() == want
        assert p.mask.cpu().numpy().nonzero()[0].tolist() == sorted(set(ids.ravel().tolist()))


@pytest.mark.parametrize("path", ["copy_engine", "sm_gather"])
def test_loads_land_in_slots(pf, path):
    E, eb = 16, 1 << 20
    store = pf.ExpertStore(E, eb)
    cache = pf.ExpertCache(8, eb, E)
    p = pf.Prefetcher(store, cache)
    ids = torch.tensor([[3, 9, 11], [9, 12, 15]], dtype=torch.int32).cuda()
    if path == "copy_engine":
        p.load_copy_engine(ids)
    else:
        p.load_sm_gather(ids)
    p.done.synchronize()
    n = int(p.need_count.item())
    lst = p.need_list[:n].cpu().tolist()
    slots = p.need_slot[:n].cpu().tolist()
    assert lst == [3, 9, 11, 12, 15]
    for e, s in zip(lst, slots):
        assert torch.equal(cache.slot(s).cpu(), store.blob(e)), (e, s)
    # residency was committed on the device by the load path itself
    assert cache.slot_of[torch.tensor(lst).cuda().long()].cpu().tolist() == slots
    assert int(cache.free_cursor.item()) == 5
    p.plan(torch.tensor([[3, 4]], dtype=torch.int32).cuda())
    torch.cuda.synchronize()
    assert p.need_list[: int(p.need_count.item())].cpu().tolist() == [4]
    assert p.need_slot[:1].cpu().tolist() == [5]   # the next free slot (device cursor)


def test_hook_point_deployment(pf):
    """SURVEY 8(f)1 (hooks.py:19,113-114; pipesim.py:272-305 executed): raw
    hidden states -> K0 RMSNorm(gamma) -> x_hat bit-identical to the oracle ->
    predicted top-m identical to the oracle's on x_hat -> those experts in the
    cache with the right bytes; after the router, exactly the missed experts
    are loaded and every true expert has a slot holding its blob."""
    import paper_2511_10676_b200 as pb
    from paper_2511_10676_b200.deploy import HookPointPredictor
    from oracle import oracle as O
    rng = np.random.default_rng(5)
    d, h, E, m, k, B = 512, 512, 32, 4, 3, 5
    model = pb.init_model("arch2", d, h, E, seed=2)
    model.w1, model.w2 = O.round_bf16(model.w1), O.round_bf16(model.w2)
    gamma = rng.uniform(0.5, 1.5, d)
    for gather in (0, 16):
        store = pf.ExpertStore(E, 8192)
        cache = pf.ExpertCache(E, 8192, E)
        hp = HookPointPredictor(model, m, "rmsnorm", gamma, prefetcher=pf.Prefetcher(store, cache), gather_ctas=gather)
        hidden = O.round_bf16(2.0 * rng.standard_normal((B, d)) + 0.3)
        x_hat, ids = hp.pre_attention(torch.from_numpy(hidden).cuda().to(torch.bfloat16))
        xo = O.input_norm_bf16(hidden, "rmsnorm", gamma)
        assert np.array_equal(x_hat.double().cpu().numpy(), xo)
        p = {"arch": "arch2", "w1": model.w1, "b1": model.b1, "w2": model.w2, "b2": model.b2}
        want = O.top_k_batch(O.predict_logits(p, xo), m)
        assert np.array_equal(ids.cpu().numpy(), want)
        hp.pf.done.synchronize()
        predicted = sorted(set(want.ravel().tolist()))
        slot_of = cache.slot_of.cpu().numpy()
        for e in predicted:
            assert slot_of[e] >= 0 and torch.equal(cache.slot(int(slot_of[e])).cpu(), store.blob(e)), e
        true = np.sort(np.stack([rng.choice(E, k, replace=False) for _ in range(B)]), axis=1)
        slots, n_emergency = hp.post_router(torch.from_numpy(true).cuda().to(torch.int32))
        torch.cuda.synchronize()
        assert n_emergency == len(set(true.ravel().tolist()) - set(predicted))
        for e, s in zip(true.ravel().tolist(), slots.cpu().numpy().ravel().tolist()):
            assert s >= 0 and torch.equal(cache.slot(int(s)).cpu(), store.blob(e)), e
        hp.check()
    bad = torch.zeros((2, d), dtype=torch.bfloat16, device="cuda")
    bad[1, 3] = float("inf")
    hp2 = HookPointPredictor(model, m, "rmsnorm", gamma)
    hp2.pre_attention(bad)
    with pytest.raises(pb.ConfigurationError):
        hp2.check()


def test_hook_point_cuda_graph(pf):
    """The captured pre_attention (HookPointPredictor.graph) gives the eager
    path's x_hat and ids on new inputs, replay after replay, and drives the
    prefetch; its launch cost is one graph replay."""
    import paper_2511_10676_b200 as pb
    from paper_2511_10676_b200.deploy import HookPointPredictor
    from oracle import oracle as O
    rng = np.random.default_rng(11)
    d, h, E, m, B = 1024, 1024, 64, 6, 3
    model = pb.init_model("arch2", d, h, E, seed=4)
    model.w1, model.w2 = O.round_bf16(model.w1), O.round_bf16(model.w2)
    gamma = rng.uniform(0.5, 1.5, d)
    store, cache = pf.ExpertStore(E, 4096), pf.ExpertCache(E, 4096, E)
    hp = HookPointPredictor(model, m, "rmsnorm", gamma, prefetcher=pf.Prefetcher(store, cache), gather_ctas=8)
    gh = hp.graph(B)
    ref = HookPointPredictor(model, m, "rmsnorm", gamma)
    for step in range(4):
        hidden = torch.from_numpy(O.round_bf16(2.0 * rng.standard_normal((B, d)))).cuda().to(torch.bfloat16)
        x_hat, ids = gh.pre_attention(hidden)
        xr, ir = ref.pre_attention(hidden, prefetch=False)
        assert torch.equal(x_hat, xr) and torch.equal(ids, ir), step
        hp.pf.done.synchronize()
        for e in set(ids.cpu().numpy().ravel().tolist()):
            s = int(cache.slot_of[e].item())
            assert s >= 0 and torch.equal(cache.slot(s).cpu(), store.blob(e)), e
    with pytest.raises(pb.ConfigurationError):
        gh.pre_attention(torch.zeros((B + 1, d), dtype=torch.bfloat16, device="cuda"))
