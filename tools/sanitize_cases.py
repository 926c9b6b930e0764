"""Small instances of every libtraj path, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_18468_b200 as P  # noqa: E402

A = np.arange(40)
for algo in ("3m", "4m"):
    P.traj_set_zgemm_algorithm(algo)
    for kw in [dict(Lx=80, protocol="projective", gammas=[4.0, 1.0]),
               dict(Lx=80, protocol="homodyne", gammas=[1.0]),
               dict(Lx=80, protocol="homodyne_rk4", gammas=[1.0]),
               dict(Lx=80, protocol="projective_events", gammas=[3.0]),
               dict(Lx=10, Ly=8, protocol="projective", gammas=[2.86]),
               dict(Lx=80, protocol="homodyne", gammas=[1.0], propagator="banded"),
               dict(Lx=80, protocol="projective", gammas=[6.0], shard_size=2)]:
        g = P.Trajectories(seed=1, **kw)
        g.step(3)
        g.entropy(A)
        g.mutual_info(np.arange(0, 10), np.arange(20, 30))
        g.particle_covariance(np.arange(0, 10), np.arange(20, 30))
        if g.Ly == 1:
            g.density_correlation(0)
        g.occupations()
        g.correlation_rows(0, 3, 5)
        g.close()
torch.cuda.synchronize()
print("sanitize cases ok")
