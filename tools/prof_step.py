"""Run trajectory steps of a config for ncu captures: --warmup steps first, then --steps steps
inside cudaProfilerStart/Stop (use ncu --profile-from-start off).  Prints nothing of value."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
import paper_2508_18468_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=0)
ap.add_argument("--traj", type=int, default=1)
a = ap.parse_args()
w = workloads.CONFIGS[a.config]()
g = [w.gamma_of(t % w.n_traj) for t in range(a.traj)]
tr = P.Trajectories(w.Lx, w.Ly, w.protocol, g, dt=w.dt, seed=w.seed)
tr.step(a.warmup)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
tr.step(a.steps)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", tr.step_index, tr.last_clicks(0))
