import sys, time, torch
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18468_b200 as P
for (Lx, Ly, g, steps) in [(16384, 1, 0.3, 10), (160, 160, 2.86, 5)]:
    tr = P.Trajectories(Lx, Ly, "projective", [g], seed=0, propagator="banded", orthonormalizer="lowrank")
    tr.step(2)
    torch.cuda.synchronize()
    s0 = tr.lowrank_stats(); c0 = tr.cqr2_fallbacks()
    t0 = time.perf_counter(); tr.step(steps); torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / steps
    s1 = tr.lowrank_stats()
    print(Lx, Ly, f"{dt*1e3:.1f} ms/step", {k: (s1[k] - s0[k]) / steps for k in s1}, "cqr2 fallbacks", tr.cqr2_fallbacks() - c0, "clicks", tr.last_clicks(0), flush=True)
    tr.close()
