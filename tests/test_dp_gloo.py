"""Data-parallel MBS logic on CPU with gloo, world_size 2 (the N>1 path's host side).

Each rank takes its block of whole micro-batches of the GLOBAL plan
(dp.partition_micro_batches), computes per-micro gradients of the same model
(torch-CPU float64, the oracle's hybrid grad fn) seeded with the GLOBAL
normalisation factors, accumulates them, and SUM-all-reduces the flat
accumulator bucket by bucket (dp.bucket_ranges) plus the loss record
(dp.combine_loss_record). The result must equal the single-process
reference-semantics mini-batch gradient and statistics.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mbs_oracle as O
from oracle.hybrid import TorchGradFn
from paper_2110_12484_b200 import dp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model():
    torch.manual_seed(3)
    return torch.nn.Sequential(torch.nn.Conv2d(3, 4, 3, padding=1), torch.nn.BatchNorm2d(4), torch.nn.ReLU(),
                               torch.nn.MaxPool2d(2), torch.nn.Flatten(), torch.nn.Linear(4 * 4 * 4, 5))


def _data(n):
    g = np.random.RandomState(0)
    return g.randn(n, 3, 8, 8), g.randint(0, 5, size=n)


def _worker(rank, world, port, n_b, n_mu, mode, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.set_num_threads(1)
        plan = O.plan_split(n_b, n_mu)
        block = dp.partition_micro_batches(plan, world)[rank]
        x, y = _data(n_b)
        gf = TorchGradFn(_model(), "cross_entropy")
        names = gf.names
        shapes = [gf.params()[n].shape for n in names]
        numels = tuple(int(np.prod(s)) for s in shapes)
        offs = np.concatenate([[0], np.cumsum(numels)])
        acc = np.zeros(offs[-1])
        losses, factors, weights = [], [], []
        for k, f in zip(range(*block), dp.local_factors(plan, block, mode)):
            lo, hi = plan.index_ranges[k]
            val, grads, _ = gf(x[lo:hi], y[lo:hi], f)
            for i, n in enumerate(names):
                acc[offs[i]:offs[i + 1]] += grads[n].ravel()
            losses.append(val)
            factors.append(f)
            weights.append(plan.sizes[k])
        t = torch.from_numpy(acc)
        for s0, s1 in dp.bucket_ranges(numels, 50):        # bucket-wise all-reduce, backward order
            dist.all_reduce(t[offs[s0]:offs[s1]])
        rec = torch.from_numpy(dp.combine_loss_record(losses, factors, weights, block, plan.n_s_mu, n_b))
        dist.all_reduce(rec)
        out_q.put((rank, t.numpy().copy(), rec.numpy().copy(), block))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_b,n_mu,mode", [(10, 4, "exact_weighted"), (16, 4, "paper_faithful"), (7, 2, "off"),
                                           (9, 9, "exact_weighted")])
def test_dp_two_ranks_equals_single_process(n_b, n_mu, mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_b, n_mu, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # every rank holds the identical reduced sum
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][2], res[1][2])
    # single-process reference semantics (engine.py:179-230)
    x, y = _data(n_b)
    gf = TorchGradFn(_model(), "cross_entropy")
    plan = O.plan_split(n_b, n_mu)
    total, st = O.mini_batch_gradient(gf, {n: v.shape for n, v in gf.params().items()}, x, y, plan, mode)
    flat = np.concatenate([total[n].ravel() for n in gf.names])
    np.testing.assert_allclose(res[0][1], flat, rtol=1e-12, atol=1e-14)
    rec = res[0][2]
    assert rec[0] == pytest.approx(st["loss"], rel=1e-12)
    np.testing.assert_allclose(rec[1:1 + plan.n_s_mu], st["losses_raw"], rtol=1e-12)
    np.testing.assert_allclose(rec[1 + plan.n_s_mu:], st["losses_normalized"], rtol=1e-12)
    assert np.sqrt(np.dot(res[0][1], res[0][1])) == pytest.approx(st["grad_norm"], rel=1e-10)


def test_partition_and_buckets():
    plan = O.plan_split(1024 * 8, 128)
    blocks = dp.partition_micro_batches(plan, 8)
    assert blocks == [(8 * r, 8 * r + 8) for r in range(8)]
    assert dp.rank_samples(plan, blocks[3]) == (3072, 4096)
    p2 = O.plan_split(256, 48)                      # [48]*5 + [16]
    b2 = dp.partition_micro_batches(p2, 4)
    assert b2 == [(0, 2), (2, 4), (4, 5), (5, 6)]
    assert [dp.rank_samples(p2, b) for b in b2] == [(0, 96), (96, 192), (192, 240), (240, 256)]
    assert dp.partition_micro_batches(O.plan_split(3, 1), 5)[-1] == (3, 3)   # idle ranks get empty blocks
    numels = (10, 200, 5, 5, 300, 1)
    br = dp.bucket_ranges(numels, 250)
    assert br[0][1] == len(numels) and br[-1][0] == 0
    covered = sorted(s for a, b in br for s in range(a, b))
    assert covered == list(range(len(numels)))
    assert dp.local_factors(p2, (5, 6), "exact_weighted") == [16 / 256]
    with pytest.raises(ValueError):
        dp.weak_scaling_plan(100, 48, 2)


def _bn_model():
    torch.manual_seed(11)
    return torch.nn.Sequential(torch.nn.Conv2d(3, 6, 3, padding=1), torch.nn.BatchNorm2d(6, momentum=0.1),
                               torch.nn.ReLU(), torch.nn.Conv2d(6, 4, 3, padding=1),
                               torch.nn.BatchNorm2d(4, momentum=0.3), torch.nn.Flatten(),
                               torch.nn.Linear(4 * 8 * 8, 5), torch.nn.BatchNorm1d(5, momentum=None))


BN_CASES = [(20, 4), (17, 3), (9, 9)]        # even split, ragged tail, one micro-batch (idle ranks)


def _bn_worker(rank, world, port, steps, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.set_num_threads(1)
        out = []
        for n_b, n_mu in BN_CASES:
            net = _bn_model().double().train()
            x = torch.from_numpy(_data(n_b * steps)[0])
            plan = O.plan_split(n_b, n_mu)
            block = dp.partition_micro_batches(plan, world)[rank]
            sync = dp.BNStatSync(net, dist)
            with torch.no_grad():
                for s in range(steps):
                    sync.snapshot()
                    for k in range(*block):
                        lo, hi = plan.index_ranges[k]
                        net(x[s * n_b + lo:s * n_b + hi])
                    sync.merge(block, plan.n_s_mu)
            out.append({k: v.clone().numpy() for k, v in net.state_dict().items() if "running" in k or "tracked" in k})
        out_q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_bn_running_stats_match_single_device():
    """DP BN running stats (momentum EMA and cumulative average) == the sequential single-device micro loop."""
    world, steps = 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bn_worker, args=(r, world, port, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for case, (n_b, n_mu) in enumerate(BN_CASES):
        net = _bn_model().double().train()
        x = torch.from_numpy(_data(n_b * steps)[0])
        plan = O.plan_split(n_b, n_mu)
        with torch.no_grad():
            for s in range(steps):
                for lo, hi in plan.index_ranges:
                    net(x[s * n_b + lo:s * n_b + hi])
        want = {k: v.numpy() for k, v in net.state_dict().items() if "running" in k or "tracked" in k}
        for _, got_all in res:
            got = got_all[case]
            assert set(got) == set(want)
            for k in want:
                np.testing.assert_allclose(got[k], want[k], rtol=1e-12, atol=1e-13, err_msg=f"{n_b}/{n_mu} {k}")


def test_bn_merge_coefficients():
    c = 0.9
    assert dp.bn_merge_coefficients(0.1, (2, 5), 8) == pytest.approx((c ** 3, c ** 3, c ** 8))
    assert dp.bn_merge_coefficients(0.1, (5, 5), 8) == pytest.approx((c ** 3, 1.0, c ** 8))
