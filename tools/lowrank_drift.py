"""Orthonormality drift of the low-rank (Loewdin) projective step without the refinement pass
(TRAJ_LOWRANK_REFINE=0): max|U^dag U - I| and ||U^dag U - I||_F every few steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2508_18468_b200 as P  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
every = int(sys.argv[3]) if len(sys.argv) > 3 else 20
gamma = float(sys.argv[4]) if len(sys.argv) > 4 else 0.3
tr = P.Trajectories(L, 1, "projective", [gamma], seed=0, propagator="banded", orthonormalizer="lowrank")
N = L // 2
G = torch.empty(N, N, dtype=torch.complex128, device="cuda")
I = torch.eye(N, dtype=torch.complex128, device="cuda")
for s in range(0, steps + 1, every):
    if s:
        tr.step(every)
    U = tr.get_state(0)
    P.traj_zgemm(1, 0, U, U, G)
    E = G - I
    print(f"L={L} step={s} max|E|={E.abs().max().item():.3e} |E|_F={torch.linalg.norm(E).item():.3e}", flush=True)
