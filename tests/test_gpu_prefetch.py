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
    p._commit_residency()
    p.plan(torch.tensor([[3, 4]], dtype=torch.int32).cuda())
    torch.cuda.synchronize()
    assert p.need_list[: int(p.need_count.item())].cpu().tolist() == [4]
