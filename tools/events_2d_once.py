"""One event window of a 96 x 96 lattice (event-driven PM, NEXT-4) between cudaProfilerStart/Stop, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2508_18468_b200 as P  # noqa: E402
Lx = int(sys.argv[1]) if len(sys.argv) > 1 else 96
tr = P.Trajectories(Lx, Lx, "projective_events", [0.3], seed=0, orthonormalizer="lowrank")
tr.step(1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
tr.step(1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("events in the window:", tr.last_clicks(0))
