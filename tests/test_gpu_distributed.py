"""The data-parallel DEVICE path under a real process group (world size 2,
two processes on the one GPU this build has, gloo all-reduces staged through
host memory; no kernel waits on another rank's kernel). Against the
single-rank run of the same data:
  * DeviceTrainer.step (fp64 mode) on a minibatch whose rows are split
    rank-strided: the all-reduced gradient within 1e-12 (relative), the loss
    equal to round-off (the batch-global normalisers, losses.py:129-130,
    214-216);
  * trainer.train with world_size 2 (fp64): parameters within 1e-10 of the
    single-rank train, the same per-epoch evaluation numbers;
  * a last minibatch with fewer rows than ranks (an empty shard) does not hang;
  * sharded DevicePredictor.evaluate: summed counters bit-identical.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _data():
    from oracle import oracle as O
    rng = np.random.default_rng(3)
    n, d, e, k = 1203, 32, 16, 2
    x = O.round_bf16(rng.standard_normal((n, d)))
    scores = O.softmax(x @ (rng.standard_normal((e, d)) / 4.0).T, axis=1).astype(np.float32)
    topk = O.top_k_batch(scores.astype(np.float64), k)
    return x.astype(np.float32), scores, topk


def _single():
    import paper_2511_10676_b200 as pb
    from paper_2511_10676_b200.losses import LossSpec
    acts, scores, topk = _data()
    m = pb.init_model("arch2", 32, 48, 16, seed=1)
    tr = pb.DeviceTrainer(m, LossSpec("ranking"), precision="fp64")
    lab = pb.BatchLabels.from_scores(torch.as_tensor(scores[:256].astype(np.float64)).cuda(), 2)
    out = tr.step(torch.as_tensor(acts[:256].astype(np.float64)).cuda(), lab.true_scores,
                  lab.topk_mask.to(torch.uint8), lab.rank_of)
    step = (float(out[0].item()), tr.grad.cpu().numpy().copy())
    cfg = pb.TrainConfig(loss=LossSpec("ranking"), hidden=48, batch_size=129, epochs=2, seed=2, precision="fp64")
    model, rep = pb.train(cfg, pb.TraceFile(32, 16, 2, acts, scores, topk))
    bf = pb.init_model("arch2", 32, 64, 16, seed=4)
    bf.w1, bf.w2 = _bf(bf.w1), _bf(bf.w2)
    dp = pb.DevicePredictor(bf)
    dp.decode_max_tokens = 0
    cnt, _, _ = dp.evaluate(torch.as_tensor(acts).cuda().to(torch.bfloat16), torch.as_tensor(topk), 2, [2, 6, 16])
    return step, (model, rep), cnt.cpu().numpy()


def _bf(a):
    from oracle import oracle as O
    return O.round_bf16(a)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_10676_b200 as pb
        from paper_2511_10676_b200.distributed import allreduce_counters_host, dp_hooks, shard_range
        from paper_2511_10676_b200.losses import LossSpec
        acts, scores, topk = _data()
        gh, lh = dp_hooks(host_staged=True)
        # one DeviceTrainer step on rank-strided rows of a 256-row minibatch
        m = pb.init_model("arch2", 32, 48, 16, seed=1)
        tr = pb.DeviceTrainer(m, LossSpec("ranking"), precision="fp64", grad_allreduce=gh, loss_allreduce=lh)
        rows = np.arange(256)[rank::world]
        lab = pb.BatchLabels.from_scores(torch.as_tensor(scores[rows].astype(np.float64)).cuda(), 2)
        out = tr.step(torch.as_tensor(acts[rows].astype(np.float64)).cuda(), lab.true_scores,
                      lab.topk_mask.to(torch.uint8), lab.rank_of, n_global=256)
        step = (float(out[0].item()), tr.grad.cpu().numpy().copy())
        # a minibatch of 1 row over 2 ranks: rank 1 has an empty shard and must still join
        r1 = np.arange(1)[rank::world]
        lab1 = pb.BatchLabels.from_scores(torch.as_tensor(scores[:1].astype(np.float64)).cuda(), 2) if len(r1) else None
        x1 = torch.as_tensor(acts[r1].astype(np.float64)).cuda().reshape(len(r1), 32)
        if lab1 is None:
            tr.step(x1, None, None, None, n_global=1)
        else:
            tr.step(x1, lab1.true_scores, lab1.topk_mask.to(torch.uint8), lab1.rank_of, n_global=1)
        # trainer.train, world size 2
        cfg = pb.TrainConfig(loss=LossSpec("ranking"), hidden=48, batch_size=129, epochs=2, seed=2,
                             precision="fp64")
        model, rep = pb.train(cfg, pb.TraceFile(32, 16, 2, acts, scores, topk), grad_allreduce=gh,
                              loss_allreduce=lh, world_size=world, rank=rank)
        # sharded evaluation
        bf = pb.init_model("arch2", 32, 64, 16, seed=4)
        bf.w1, bf.w2 = _bf(bf.w1), _bf(bf.w2)
        dp = pb.DevicePredictor(bf)
        dp.decode_max_tokens = 0
        lo, hi = shard_range(len(acts), rank, world)
        cnt, _, _ = dp.evaluate(torch.as_tensor(acts[lo:hi]).cuda().to(torch.bfloat16),
                                torch.as_tensor(topk[lo:hi]), 2, [2, 6, 16])
        allreduce_counters_host(cnt)
        if rank == 0:
            q.put(("ok", step, (model.w1, model.b1, model.w2, model.b2,
                                [(r.train_loss, r.exact_match, r.top1, r.overprov) for r in rep.epochs]),
                   cnt.cpu().numpy()))
    except Exception as exc:  # surface the worker's error in the test
        q.put(("error", repr(exc), None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_dp_device_path_world2():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, step, trained, cnt = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", step
    (loss1, grad1), (model1, rep1), cnt1 = _single()
    loss2, grad2 = step
    assert loss2 == pytest.approx(loss1, rel=1e-13)
    assert np.allclose(grad2, grad1, rtol=1e-12, atol=1e-14 * np.abs(grad1).max())
    w1, b1, w2, b2, rows = trained
    for a, b in ((w1, model1.w1), (b1, model1.b1), (w2, model1.w2), (b2, model1.b2)):
        assert np.allclose(a, b, rtol=1e-10, atol=1e-12)
    for r, e in zip(rows, rep1.epochs):
        assert r[0] == pytest.approx(e.train_loss, rel=1e-10)
        assert r[1:] == (e.exact_match, e.top1, e.overprov)
    assert np.array_equal(cnt, cnt1)
