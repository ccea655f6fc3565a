"""DataParallelMBS on the GPU: 2 ranks sharing cuda:0 (gloo carries CUDA tensors), and 1-rank NCCL.

The run's GPU allocation is a single B200, so two ranks share it; the
data-parallel step (global plan partition, global factors, bucketed K1 from
post-accumulate-grad hooks with async all-reduce, reduced-norm guard, K3)
must reproduce the single-process MBS mini-batch: identical loss record and
post-step weights to fp32 summation-order rounding.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _net():
    torch.manual_seed(5)
    return torch.nn.Sequential(torch.nn.Conv2d(3, 16, 3, padding=1), torch.nn.BatchNorm2d(16), torch.nn.ReLU(),
                               torch.nn.Conv2d(16, 16, 3, padding=1), torch.nn.ReLU(), torch.nn.MaxPool2d(2),
                               torch.nn.Flatten(), torch.nn.Linear(16 * 4 * 4, 7))


def _data(n):
    g = torch.Generator().manual_seed(9)
    return torch.randn(n, 3, 8, 8, generator=g), torch.randint(0, 7, (n,), generator=g)


def _rank(rank, world, port, backend, n_per_rank, n_mu, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        import paper_2110_12484_b200 as mbs
        from paper_2110_12484_b200.dp import DataParallelMBS
        dev = torch.device("cuda:0")
        net = _net().to(dev)
        params = mbs.ParameterSet(net)
        x, y = _data(n_per_rank * world)
        xs, ys = x[rank * n_per_rank:(rank + 1) * n_per_rank], y[rank * n_per_rank:(rank + 1) * n_per_rank]
        d = DataParallelMBS(params, bucket_mb=0.002)      # tiny buckets: several all-reduces per step
        st = mbs.sgd_state(0.05, 0.9, 5e-4)
        acc = mbs.GradientAccumulator(params)
        out = []
        for step in range(2):
            r = d.train_mini_batch(net, (xs.to(dev), ys.to(dev)), n_per_rank, n_mu, mode, "cross_entropy", st,
                                   accumulator=acc)
            out.append((r.loss, list(r.losses_raw), r.grad_norm, r.step_count))
        q.put((rank, params.flat.cpu().numpy().copy(), out, len(d.buckets), _bn_state(net)))
    finally:
        dist.destroy_process_group()


def _bn_state(net):
    return {k: v.detach().cpu().double().numpy().copy() for k, v in net.state_dict().items()
            if "running" in k or "tracked" in k}


def _single(n_b, n_mu, mode, steps=2, with_bn=False):
    import paper_2110_12484_b200 as mbs
    torch.backends.cudnn.allow_tf32 = False
    dev = torch.device("cuda:0")
    net = _net().to(dev)
    params = mbs.ParameterSet(net)
    x, y = _data(n_b)
    st = mbs.sgd_state(0.05, 0.9, 5e-4)
    out = []
    acc = mbs.GradientAccumulator(params)
    for step in range(steps):
        _, s = mbs.train_mini_batch(net, params, (x.to(dev), y.to(dev)), mbs.plan_split(n_b, n_mu), mode,
                                    "cross_entropy", st, accumulator=acc)
        out.append((s.loss, list(s.losses_raw), s.grad_norm, s.step_count))
    if with_bn:
        return params.flat.cpu().numpy(), out, _bn_state(net)
    return params.flat.cpu().numpy(), out


def _run(world, backend, n_per_rank, n_mu, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, backend, n_per_rank, n_mu, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("mode", ["exact_weighted", "paper_faithful"])
def test_two_ranks_share_one_gpu_gloo(cuda, mode):
    n_per_rank, n_mu = 12, 4
    res = _run(2, "gloo", n_per_rank, n_mu, mode)
    assert res[0][3] > 1
    np.testing.assert_array_equal(res[0][1], res[1][1])           # every rank steps identically
    w_single, out_single, bn_single = _single(2 * n_per_rank, n_mu, mode, with_bn=True)
    err = np.linalg.norm(res[0][1] - w_single) / np.linalg.norm(w_single)
    assert err <= 1e-6, err
    # BN running statistics merged by BNStatSync == the single-device sequential micro loop (fp32 rounding)
    for k, v in bn_single.items():
        for r in range(2):
            np.testing.assert_allclose(res[r][4][k], v, rtol=1e-5, atol=1e-6, err_msg=k)
    for (l, raw, gn, sc), (l1, raw1, gn1, sc1) in zip(res[0][2], out_single):
        assert sc == sc1
        assert l == pytest.approx(l1, rel=1e-5)
        np.testing.assert_allclose(raw, raw1, rtol=1e-5)
        assert gn == pytest.approx(gn1, rel=1e-5)


def test_one_rank_nccl(cuda):
    res = _run(1, "nccl", 12, 4, "exact_weighted")
    w_single, out_single = _single(12, 4, "exact_weighted")
    err = np.linalg.norm(res[0][1] - w_single) / np.linalg.norm(w_single)
    assert err <= 1e-6, err


def _rank_peer(rank, world, port, n_per_rank, n_mu, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2110_12484_b200 as mbs
        from paper_2110_12484_b200.dp import DataParallelMBS
        dev = torch.device("cuda:0")
        net = _net().to(dev)
        params = mbs.ParameterSet(net)
        x, y = _data(n_per_rank * world)
        xs, ys = x[rank * n_per_rank:(rank + 1) * n_per_rank], y[rank * n_per_rank:(rank + 1) * n_per_rank]
        d = DataParallelMBS(params, transport="peer")
        st = mbs.sgd_state(0.05, 0.9, 5e-4)
        acc = mbs.GradientAccumulator(params)
        out = []
        for step in range(3):
            r = d.train_mini_batch(net, (xs.to(dev), ys.to(dev)), n_per_rank, n_mu, mode, "cross_entropy", st,
                                   accumulator=acc)
            out.append((r.loss, list(r.losses_raw), r.grad_norm, r.step_count))
        torch.cuda.synchronize()
        assert not d.peer.error()
        q.put((rank, params.flat.cpu().numpy().copy(), out, acc.flat.cpu().numpy().copy()))
        dist.barrier()
        d.peer.close()
    finally:
        dist.destroy_process_group()


def test_fused_peer_allreduce_two_ranks_one_gpu(cuda):
    """K1C: last-micro accumulate + all-reduce in one kernel over CUDA-IPC peer memory (2 ranks, 1 GPU)."""
    n_per_rank, n_mu, mode = 12, 4, "exact_weighted"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_peer, args=(r, 2, port, n_per_rank, n_mu, mode, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(res[0][1], res[1][1])       # identical weights on both ranks
    np.testing.assert_array_equal(res[0][3], res[1][3])       # identical reduced accumulators
    w_single, out_single = _single(2 * n_per_rank, n_mu, mode, steps=3)
    err = np.linalg.norm(res[0][1] - w_single) / np.linalg.norm(w_single)
    assert err <= 1e-6, err
    for (l, raw, gn, sc), (l1, raw1, gn1, sc1) in zip(res[0][2], out_single):
        assert sc == sc1
        assert l == pytest.approx(l1, rel=1e-5)
        np.testing.assert_allclose(raw, raw1, rtol=1e-5)
        assert gn == pytest.approx(gn1, rel=1e-5)


def _rank_epoch(rank, world, port, shard, mini, n_mu, q, transport):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2110_12484_b200 as mbs
        from paper_2110_12484_b200.dp import DataParallelMBS
        dev = torch.device("cuda:0")
        net = _net().to(dev)
        params = mbs.ParameterSet(net)
        x, y = _data(shard * world)
        xs, ys = x[rank * shard:(rank + 1) * shard], y[rank * shard:(rank + 1) * shard]
        d = DataParallelMBS(params, transport=transport)
        st = mbs.sgd_state(0.05, 0.9, 5e-4)
        acc = mbs.GradientAccumulator(params)
        res = d.train_epoch(net, xs, ys, mini_batch_size=mini, micro_batch_size=n_mu,
                            normalization="exact_weighted", loss_kind="cross_entropy", optimizer_state=st, seed=4,
                            epoch_index=1, accumulator=acc, prefetch=True)      # host shard: streamed
        q.put((rank, params.flat.cpu().numpy().copy(), [r.loss for r in res], st.step_count))
        dist.barrier()
        if d.peer is not None:
            d.peer.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_dp_train_epoch_weak_scaling(cuda, transport):
    """Each rank streams its own host shard in its own order; == single process on the united mini-batches."""
    import paper_2110_12484_b200 as mbs
    world, shard, mini, n_mu = 2, 24, 12, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_epoch, args=(r, world, port, shard, mini, n_mu, q, transport))
          for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(res[0][1], res[1][1])
    assert res[0][3] == shard // mini
    # single process: global mini-batch m = concat_r shard_r[order_r[m*mini:(m+1)*mini]]
    x, y = _data(shard * world)
    orders = [mbs.named_stream(4, f"shuffle/epoch1/rank{r}").permutation(shard) for r in range(world)]
    dev = torch.device("cuda:0")
    net = _net().to(dev)
    params = mbs.ParameterSet(net)
    st = mbs.sgd_state(0.05, 0.9, 5e-4)
    acc = mbs.GradientAccumulator(params)
    losses = []
    for m in range(shard // mini):
        idx = np.concatenate([r * shard + orders[r][m * mini:(m + 1) * mini] for r in range(world)])
        ii = torch.from_numpy(idx.astype(np.int64))
        _, s = mbs.train_mini_batch(net, params, (x[ii].to(dev), y[ii].to(dev)),
                                    mbs.plan_split(world * mini, n_mu), "exact_weighted", "cross_entropy", st,
                                    accumulator=acc)
        losses.append(s.loss)
    w = params.flat.cpu().numpy()
    assert np.linalg.norm(res[0][1] - w) / np.linalg.norm(w) <= 1e-6
    np.testing.assert_allclose(res[0][2], losses, rtol=1e-5)
