"""One banded+low-rank c3 step and one chol_inverse(8192) for ncu captures of the small kernels
(banded_kernel, probe_*, chol_leaf_kernel).  Not a timing tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2508_18468_b200 as P  # noqa: E402

tr = P.Trajectories(16384, 1, "projective", [0.3], seed=0, propagator="banded", orthonormalizer="lowrank")
tr.step(2)
torch.cuda.synchronize()
tr.close()
