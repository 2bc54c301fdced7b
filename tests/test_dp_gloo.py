"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel host logic: rank ->
worker/stream plan, the all-reduce mean of per-rank gradients, and exact pooled statistics,
against the oracle's L-worker trainer (proj/src/trainer.cpp:111-306)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, workers_per_rank):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    import pyoracle as O
    from paper_2106_13308_b200 import dp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, mbs, seed = 8, 64, 11
    e = O.random_maxcut_graph(n, 3)
    m = O.made_init(n, 8, seed)
    plan = dp.RankPlan(rank, world, workers_per_rank)
    # this rank's workers: same streams as the reference's workers first_worker .. +L_r
    g_sum = np.zeros(m.d)
    cs = cq = 0
    for s in plan.streams():
        x, _ = O.auto_sample(m, mbs, seed=seed, stream=s)
        le, cut = O.local_energy(n, e, x)
        g_sum += O.gradient_from_locals(m, x, le)
        cs += int(cut.sum())
        cq += int((cut.astype(np.int64) ** 2).sum())
    t = torch.tensor(g_sum)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)  # the step's one collective (NCCL sum on the GPU)
    g = t.numpy() * plan.grad_scale
    cs, cq = dp.allreduce_sums([cs, cq])
    mean, var = dp.pooled_stats(len(e), plan.total_workers * mbs, cs, cq)
    uid = dp.share_unique_id(bytes([7] * 128) if rank == 0 else bytes(128))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), g=g, mean=mean, var=var, uid=np.frombuffer(uid, np.uint8))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,wpr", [(2, 1), (2, 2)])
def test_dp_two_ranks_match_reference_workers(tmp_path, world, wpr):
    import pyoracle as O
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path), wpr), nprocs=world, join=True,
                       start_method="spawn")
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(world)]
    L = world * wpr
    ref = O.train(8, O.random_maxcut_graph(8, 3), h=8, optimizer="sgd", iterations=1, workers=L, minibatch=64,
                  eval_batch=16, seed=11, want_first_grad=True)
    for k in range(world):
        # replicas see the identical reduced gradient; equal to the tree mean up to fp64 order
        assert np.array_equal(r[k]["g"], r[0]["g"])
        assert np.abs(r[k]["g"] - ref["first_grad"]).max() <= 1e-12
        # pooled statistics: bit-exact with the reference's two-pass fp64 over L*mbs energies
        assert r[k]["mean"] == ref["stats"][0, 0]
        assert np.sqrt(r[k]["var"]) == ref["stats"][0, 1]
        assert bytes(r[k]["uid"]) == bytes([7] * 128)


def test_rank_plan_streams():
    from paper_2106_13308_b200 import dp
    p = dp.RankPlan(rank=3, world=8, workers_per_rank=2)
    assert p.streams() == [7, 8] and p.total_workers == 16 and p.grad_scale == 1 / 16
