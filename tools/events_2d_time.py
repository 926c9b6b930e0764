"""Event-driven PM (NEXT-4) on a 2d lattice: ms per event pass, separable (default) against the
product taps in one kernel (TRAJ_EV_SEPARABLE=0).  python tools/events_2d_time.py [Lx] [gamma] [windows]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2508_18468_b200 as P  # noqa: E402

Lx = int(sys.argv[1]) if len(sys.argv) > 1 else 96
gam = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
windows = int(sys.argv[3]) if len(sys.argv) > 3 else 3
for sep in ("1", "0"):
    os.environ["TRAJ_EV_SEPARABLE"] = sep
    tr = P.Trajectories(Lx, Lx, "projective_events", [gam], seed=0, orthonormalizer="lowrank")
    tr.step(1)
    torch.cuda.synchronize()
    ev = 0
    t0 = time.perf_counter()
    for _ in range(windows):
        tr.step(1)
        ev += tr.last_clicks(0)[0]
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    L, N = Lx * Lx, Lx * Lx // 2
    gb = 2.0 * L * N * 16 / 1e9
    print(f"{Lx}x{Lx} gamma={gam} TRAJ_EV_SEPARABLE={sep}: {windows} windows, {ev} events, {ms / windows:.1f} ms/window, "
          f"{ms / max(ev + windows, 1):.3f} ms per pass (one read + one write of U = {gb:.2f} GB -> "
          f"{gb / (ms / max(ev + windows, 1) / 1e3):.0f} GB/s algorithmic)")
    del tr
