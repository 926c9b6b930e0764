"""Debug driver (round 2): projective steps through the C-ABI vs the oracle, step by step, under
environment variants passed as KEY=VAL arguments.  Prints one line per step."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for kv in sys.argv[4:]:
    k, v = kv.split("=")
    os.environ[k] = v

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_18468_b200 as P  # noqa: E402
from oracle import lattice  # noqa: E402
from oracle.trajectory import OracleTrajectory  # noqa: E402

L, gamma, steps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
P.load_library()
g = P.Trajectories(L, 1, "projective", [gamma], seed=11)
o = OracleTrajectory(L, 1, "projective", gamma, 0.05, seed=11, traj=0, K=lattice.propagator_lattice(L, 1, 1.0, 0.05))
for s in range(steps):
    g.step(1)
    o.step(1)
    U = g.get_state(0)
    nan = bool(torch.isnan(U).any().item())
    C = g.correlation(0).cpu().numpy()
    dC = float(np.abs(C - o.correlation()).max())
    G = (U.conj().T @ U).cpu().numpy()
    print(f"L={L} step {s}: clicks gpu {g.last_clicks(0)} oracle {(o.last_clicks[0].size, int(o.last_clicks[1].sum()))} "
          f"nan={nan} dC={dC:.2e} orth={np.abs(G - np.eye(G.shape[0])).max():.2e} fb={g.cqr2_fallbacks()} "
          f"env={sys.argv[4:]}", flush=True)
