"""Time traj_chol_inverse for small n per Cholesky leaf (TRAJ_CHOL_LEAF=blk|elim|regs), CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_18468_b200 as P  # noqa: E402
from paper_2508_18468_b200 import traj_chol_inverse  # noqa: E402

P.load_library()
for n in (64, 128, 1024, 8192):
    rng = np.random.default_rng(n)
    M = rng.standard_normal((n + 9, n)) + 1j * rng.standard_normal((n + 9, n))
    G0 = torch.from_numpy(M.conj().T @ M).cuda()
    for leaf in ("blk", "elim", "regs"):
        os.environ["TRAJ_CHOL_LEAF"] = leaf
        X = torch.zeros((n, n), dtype=torch.complex128, device="cuda")
        G = G0.clone()
        traj_chol_inverse(G, X)
        reps = 50 if n <= 1024 else 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            G.copy_(G0)
            traj_chol_inverse(G, X)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        R = np.linalg.cholesky(G0.cpu().numpy()).conj().T
        err = np.abs(X.cpu().numpy() @ R - np.eye(n)).max()
        print(f"n={n:5d} leaf={leaf:5s} {ms * 1e3:10.1f} us  |X R - I| = {err:.1e}", flush=True)
