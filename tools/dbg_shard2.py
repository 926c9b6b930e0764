"""Debug driver (round 2): sharded-emulation projective steps vs the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for kv in sys.argv[4:]:
    k, v = kv.split("=")
    os.environ[k] = v
os.environ["TRAJ_DEBUG_SHARD"] = "1"
import numpy as np  # noqa: E402
import paper_2508_18468_b200 as P  # noqa: E402
from oracle import lattice  # noqa: E402
from oracle.trajectory import OracleTrajectory  # noqa: E402

L, shards, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
P.load_library()
g = P.Trajectories(L, 1, "projective", [4.0], seed=13, traj_base=2, shard_size=shards)
o = OracleTrajectory(L, 1, "projective", 4.0, 0.05, seed=13, traj=2, K=lattice.propagator_lattice(L, 1, 1.0, 0.05))
for s in range(steps):
    g.step(1)
    o.step(1)
    C = g.correlation(0).cpu().numpy()
    print(f"step {s}: gpu {g.last_clicks(0)} oracle {(o.last_clicks[0].size, int(o.last_clicks[1].sum()))} "
          f"dC {np.abs(C - o.correlation()).max():.2e} env {sys.argv[4:]}", flush=True)
