"""Host logic of the trajectory-parallel path on CPU: world_size-2 gloo process groups
(127.0.0.1), the id partition and the one-collective moment reduction."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_18468_b200.ensemble import accumulate, allreduce_sums, moments_to_stats, partition


@pytest.mark.parametrize("n,world", [(1, 1), (16, 2), (17, 2), (192, 8), (5, 8), (256, 3)])
def test_partition_covers_each_id_once(n, world):
    seen = []
    for r in range(world):
        s, c = partition(n, world, r)
        seen.extend(range(s, s + c))
    assert seen == list(range(n))


def test_moments_to_stats():
    x = np.array([0.3, 0.9, 1.4, 2.2])
    sums = np.array([x.sum(), (x * x).sum(), x.size])
    m, e, n = moments_to_stats(sums)
    assert m == pytest.approx(x.mean())
    assert e == pytest.approx(x.std(ddof=1) / np.sqrt(x.size))
    assert n == 4


def test_accumulate_excludes_failed_and_groups_by_gamma():
    vals = np.array([1.0, 2.0, np.nan, 4.0])
    ok = np.array([True, False, True, True])
    g = np.array([0, 0, 1, 1])
    out = accumulate(vals, ok, g, 2)
    assert np.allclose(out, [[1, 1, 1], [4, 16, 1]])


def _worker(rank, world, port, n_traj, n_times, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    allv = rng.random((n_traj, n_times))          # the same synthetic per-trajectory values on every rank
    s, c = partition(n_traj, world, rank)
    local = np.zeros((n_times, 2, 3))
    for k in range(n_times):
        local[k] = accumulate(allv[s:s + c, k], np.ones(c, bool), np.arange(s, s + c) % 2, 2)
    tot = allreduce_sums(local)
    q.put((rank, tot))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_reduction_matches_global_statistics():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    world, n_traj, n_times = 2, 13, 4
    ps = [ctx.Process(target=_worker, args=(r, world, port, n_traj, n_times, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(res[0], res[1])
    allv = np.random.default_rng(0).random((n_traj, n_times))
    m, e, n = moments_to_stats(res[0])
    for k in range(n_times):
        for g in range(2):
            x = allv[g::2, k]
            assert n[k, g] == x.size
            assert m[k, g] == pytest.approx(x.mean(), rel=1e-12)
            assert e[k, g] == pytest.approx(x.std(ddof=1) / np.sqrt(x.size), rel=1e-9)
