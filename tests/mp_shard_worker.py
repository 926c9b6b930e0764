"""Worker of tests/test_gpu_multirank.py (launched by torch.distributed.run, one rank per GPU):
one trajectory row-sharded over the ranks through NCCL, checked on rank 0 against the oracle and
against the single-GPU emulation of the same shard count.  Prints one JSON line on rank 0."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    L, Ly, protocol, gamma, steps, propagator = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3],
                                                 float(sys.argv[4]), int(sys.argv[5]), sys.argv[6])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2508_18468_b200 as P
    P.load_library()
    box = [P.traj_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    Lx = L // Ly
    tr = P.Trajectories(Lx, Ly, protocol, [gamma], seed=3, shard_size=world, shard_rank=rank, nccl_id=box[0],
                        propagator=propagator)
    tr.step(steps)
    C = tr.correlation(0).cpu().numpy()          # allgathers U: every rank holds the full C
    A = np.arange(L // 2) if Ly == 1 else np.nonzero(np.arange(L) % Lx < Lx // 2)[0]
    S = tr.entropy(A)[0]
    clicks = tr.last_clicks(0)
    tr.close()
    out = {}
    if rank == 0:
        from oracle import lattice
        from oracle.trajectory import OracleTrajectory
        o = OracleTrajectory(Lx, Ly, protocol, gamma, 0.05, seed=3, traj=0,
                             K=lattice.propagator_lattice(Lx, Ly, 1.0, 0.05))
        o.step(steps)
        em = P.Trajectories(Lx, Ly, protocol, [gamma], seed=3, shard_size=world, propagator=propagator)
        em.step(steps)
        out = {"dC_oracle": float(np.abs(C - o.correlation()).max()), "dS_oracle": float(abs(S - o.entropy(A))),
               "dC_emulation": float(np.abs(C - em.correlation(0).cpu().numpy()).max()),
               "clicks": list(clicks), "clicks_emulation": list(em.last_clicks(0)),
               "clicks_oracle": [int(o.last_clicks[0].size), int(o.last_clicks[1].sum())]
               if protocol == "projective" else list(clicks)}
        em.close()
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
