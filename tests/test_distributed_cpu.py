"""Multi-process (gloo, world_size 2) tests of the sharding scheme on CPU.

* evaluation: per-rank counters on contiguous token shards, summed with
  allreduce_counters, equal the single-process counters bit for bit;
* training: rank-strided minibatch slices with the loss partial sums
  all-reduced before the global normalisers reproduce the full-batch loss and
  gradient (the data-parallel contract of trainer.train / DeviceTrainer).
Arithmetic uses the oracle (CPU); the device kernels implement the same
partial-sum layout (moep_loss partials, counter partials).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_10676_b200.distributed import allreduce_counters, dp_hooks, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _counter_vec(c, e):
    ms = c["m_values"]
    return np.concatenate([[c["n"], c["top1_count"]], [c["overprov_count"][m] for m in ms],
                           [c["recall_count"][m] for m in ms], c["per_expert_hits"], c["per_expert_truth"]])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    rng = np.random.default_rng(0)
    n, e, k = 1001, 64, 6
    z = rng.standard_normal((n, e))
    z[::5, 3] = z[::5, 4]
    truth = np.sort(rng.permuted(np.tile(np.arange(e), (n, 1)), axis=1)[:, :k], axis=1)
    lo, hi = shard_range(n, rank, world)
    c = torch.as_tensor(_counter_vec(O.eval_counters(z[lo:hi], truth[lo:hi], e), e).astype(np.int64))
    allreduce_counters(c)
    full = _counter_vec(O.eval_counters(z, truth, e), e)
    ok_counters = np.array_equal(c.numpy(), full)

    # training normalisers: rank-strided rows of one minibatch
    scores = O.softmax(rng.standard_normal((64, 16)), axis=1)
    zz = rng.standard_normal((64, 16))
    lab = O.batch_labels(scores, 2)
    rows = np.arange(64)[rank::world]
    sub = {kk: v[rows] for kk, v in lab.items()}
    # unnormalised parts, as the K4 partials: bce (already / N_global*E), hinge total, n_pairs
    w = O.tier_weights(sub, 3.0, 0.5, 1.5)
    t = sub["topk_mask"]
    logs = np.where(t, -np.logaddexp(0, -zz[rows]), -np.logaddexp(0, zz[rows]))
    bce = -np.sum(w * logs) / (64 * 16)
    hinge, ghinge, npairs = O.ranking_hinge(zz[rows], sub, normalize=False)
    parts = torch.tensor([bce, hinge, float(npairs)], dtype=torch.float64)
    _, loss_ar = dp_hooks()
    loss_ar(parts)
    loss = parts[0].item() + 0.3 * parts[1].item() / parts[2].item()
    ref_loss, ref_grad = O.loss_and_grad({"family": "ranking"}, zz, lab)
    g_bce = w * (O.sigmoid(zz[rows]) - t) / (64 * 16)
    g_local = g_bce + 0.3 * ghinge / parts[2].item()
    ok_loss = abs(loss - ref_loss) <= 1e-12 * abs(ref_loss)
    ok_grad = np.allclose(g_local, ref_grad[rows], rtol=1e-12, atol=1e-15)
    q.put((rank, ok_counters, ok_loss, ok_grad))
    dist.destroy_process_group()


def test_gloo_world2_sharding_contract():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_c, ok_l, ok_g in res:
        assert ok_c, f"rank {rank}: sharded counters differ"
        assert ok_l, f"rank {rank}: DP loss differs from full batch"
        assert ok_g, f"rank {rank}: DP gradient slice differs from full batch"


@pytest.mark.parametrize("n,world", [(10, 3), (1, 2), (1 << 20, 8), (7, 8)])
def test_shard_range_partitions(n, world):
    spans = [shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1
