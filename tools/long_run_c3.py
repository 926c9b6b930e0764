"""Full-size stability run: c3 (L = 16384, projective gamma = 0.3) for many steps on the default
(planar) path; every `every` steps: max |U^dag U - I|, particle number, failures, CQR2 fallbacks,
S_A(L/8).  Usage: python tools/long_run_c3.py [steps] [every]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2508_18468_b200 as P  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
every = int(sys.argv[2]) if len(sys.argv) > 2 else 50
L, N = 16384, 8192
tr = P.Trajectories(L, 1, "projective", [0.3], dt=0.05, seed=0)
G = torch.empty(N, N, dtype=torch.complex128, device="cuda")
I = torch.eye(N, dtype=torch.complex128, device="cuda")
t0 = time.time()
for s in range(every, steps + 1, every):
    tr.step(every)
    U = tr.get_state(0)
    P.traj_zgemm(1, 0, U, U, G)
    dev = (G - I).abs().max().item()
    del U
    n = tr.occupations()[0].sum().item()
    S = tr.entropy(np.arange(L // 8))[0]
    print(f"step {s}: max|U^dag U - I| = {dev:.2e}  sum n = {n:.10f}  failed = {tr.failed(0)}  "
          f"cqr2 fallbacks = {tr.cqr2_fallbacks()}  S(L/8) = {S:.6f}  clicks = {tr.last_clicks(0)}  "
          f"[{time.time() - t0:.0f} s]", flush=True)
