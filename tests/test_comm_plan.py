"""Host logic of the row-sharded step's communication, on CPU.

The NCCL executor in csrc/shard.cu issues exactly the schedules ``traj_comm_plan`` exports
(csrc/comm_plan.h).  Here they are checked without GPUs:

- every rank's list, matched under NCCL's rule -- the operations between one pair of ranks pair up
  in issue order -- puts on each receive the block that receive names, with no deadlock across the
  groups (event simulation of group-by-group progress), for P = 1..8;
- the distributed Cholesky's broadcasts are the same sequence on every rank and the slices of each
  split GEMM partition its rows;
- the ring and halo schedules, run with real message passing (torch.distributed gloo send/recv,
  world sizes 2 and 4, 127.0.0.1), deliver every rank the data of the ranks the plan names.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SEND, RECV = 0, 1


@pytest.fixture(scope="module")
def P():
    from paper_2508_18468_b200 import build
    build.build()
    import paper_2508_18468_b200 as P
    P.load_library()
    return P


def simulate(plans):
    """NCCL semantics: each rank posts its groups in order; an op pairs with the first unpaired op
    of the opposite kind between the same two ranks (issue order); a group completes when all its
    ops are paired.  Returns the pairs (sender, send op, receiver, recv op); asserts progress."""
    Pn = len(plans)
    groups = []
    for r in range(Pn):
        g = {}
        for i, op in enumerate(plans[r]):
            g.setdefault(int(op[0]), []).append(i)
        groups.append([g[k] for k in sorted(g)])
    pos = [0] * Pn                       # current group per rank
    posted = {}                          # (src, dst, kind) -> unpaired (rank, op index), issue order
    seen = set()
    paired = [set() for _ in range(Pn)]
    pairs = []
    progress = True
    while progress:
        progress = False
        for r in range(Pn):
            if pos[r] >= len(groups[r]):
                continue
            for i in groups[r][pos[r]]:
                key = (r, i)
                if key in seen:
                    continue
                seen.add(key)
                op = plans[r][i]
                src, dst = (r, int(op[2])) if op[1] == SEND else (int(op[2]), r)
                posted.setdefault((src, dst, int(op[1])), []).append(key)
        for (src, dst, kind), lst in list(posted.items()):
            if kind != SEND:
                continue
            rl = posted.get((src, dst, RECV), [])
            while lst and rl:
                s, rv = lst.pop(0), rl.pop(0)
                paired[s[0]].add(s[1])
                paired[rv[0]].add(rv[1])
                pairs.append((s[0], plans[s[0]][s[1]], rv[0], plans[rv[0]][rv[1]]))
                progress = True
        for r in range(Pn):
            while pos[r] < len(groups[r]) and all(i in paired[r] for i in groups[r][pos[r]]):
                pos[r] += 1
                progress = True
    assert all(pos[r] == len(groups[r]) for r in range(Pn)), "deadlock: a group never completes"
    return pairs


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("Pn", [1, 2, 3, 4, 5, 8])
def test_plans_pair_under_nccl_issue_order(P, kind, Pn):
    plans = [P.traj_comm_plan(kind, Pn, r) for r in range(Pn)]
    if Pn == 1 and kind == 0:
        assert plans[0].shape[0] == 0
        return
    pairs = simulate(plans)
    assert len(pairs) == sum((p[:, 1] == SEND).sum() for p in plans)
    for s, sop, r, rop in pairs:
        assert sop[4] == rop[4], (kind, Pn, s, r, sop, rop)     # the block sent is the block expected
    if kind == 0:
        # every rank receives every other rank's block exactly once, in ring-distance order
        for r in range(Pn):
            got = [int(op[4]) for op in plans[r] if op[1] == RECV]
            assert got == [(r - d) % Pn for d in range(1, Pn)]
    else:
        for r in range(Pn):
            recv = {int(op[3]): int(op[4]) for op in plans[r] if op[1] == RECV}
            assert recv == {0: 2 * ((r - 1) % Pn) + 1, 1: 2 * ((r + 1) % Pn)}


@pytest.mark.parametrize("n", [2048, 8192, 12800])
@pytest.mark.parametrize("Pn", [2, 4, 8])
def test_distributed_cholesky_broadcasts_agree(P, n, Pn):
    plans = [P.traj_comm_plan(2, Pn, r, n) for r in range(Pn)]
    for p in plans[1:]:
        assert np.array_equal(p, plans[0])
    assert plans[0].shape[0] > 0
    assert set(plans[0][:, 0]) <= set(range(Pn))
    assert (plans[0][:, 1] > 0).all() and (plans[0][:, 1] % 128 == 0).sum() >= plans[0].shape[0] - 4 * 8


def test_distributed_cholesky_slices_partition():
    from math import sqrt
    for M in (1024, 2048, 4096, 6400, 8192):
        for Pn in (2, 3, 4, 8):
            for tri in (False, True):
                # comm_plan.h row_slices, restated: 128-aligned cuts at i/P of the rows (or of the
                # triangle's area), monotone, covering [0, M)
                b = [0]
                for i in range(1, Pn):
                    f = i / Pn
                    x = M * (1 - sqrt(1 - f)) if tri else M * f
                    b.append(min(M, max(b[-1], int(x / 128.0 + 0.5) * 128)))
                b.append(M)
                assert all(b[i] <= b[i + 1] for i in range(Pn)) and b[0] == 0 and b[-1] == M


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2508_18468_b200 as P
    P.load_library()
    out = {}
    # ring exchange of the propagate: own block = rank id in every entry
    plan = P.traj_comm_plan(0, world, rank)
    own = torch.full((16,), float(rank))
    recv = {}
    for grp in sorted(set(plan[:, 0].tolist())):
        ops = []
        for op in plan[plan[:, 0] == grp]:
            if op[1] == SEND:
                ops.append(dist.P2POp(dist.isend, own, int(op[2])))
            else:
                buf = torch.empty(16)
                recv[int(op[4])] = buf
                ops.append(dist.P2POp(dist.irecv, buf, int(op[2])))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    out["ring"] = {b: float(v[0]) for b, v in recv.items() if torch.all(v == v[0])}
    # halo exchange: low edge = 2 rank, high edge = 2 rank + 1
    plan = P.traj_comm_plan(1, world, rank)
    edges = [torch.full((8,), float(2 * rank)), torch.full((8,), float(2 * rank + 1))]
    halos = [torch.empty(8), torch.empty(8)]
    ops = []
    for op in plan:
        if op[1] == SEND:
            ops.append(dist.P2POp(dist.isend, edges[int(op[3])], int(op[2])))
        else:
            ops.append(dist.P2POp(dist.irecv, halos[int(op[3])], int(op[2])))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    out["halo"] = [float(h[0]) for h in halos]
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_runs_the_schedules(P, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() + world) % 1000
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r]["ring"] == {b: float(b) for b in range(world) if b != r}
        assert res[r]["halo"] == [2 * ((r - 1) % world) + 1, 2 * ((r + 1) % world)]


def test_simulation_rejects_broken_schedules(P):
    """The checker itself: a halo plan whose two sends are swapped on one rank delivers the wrong
    edges with P = 2 (left == right), and a ring plan whose groups run in the opposite order on one
    rank deadlocks with P = 3."""
    plans = [P.traj_comm_plan(1, 2, r).copy() for r in range(2)]
    plans[0][[0, 1]] = plans[0][[1, 0]]
    assert any(s[4] != r[4] for _, s, _, r in simulate(plans))
    plans = [P.traj_comm_plan(0, 3, r).copy() for r in range(3)]
    plans[0][:, 0] = 1 - plans[0][:, 0]
    with pytest.raises(AssertionError, match="deadlock"):
        simulate(plans)
