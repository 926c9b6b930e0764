"""Two event windows of c3 with the low-rank orthonormaliser (for launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2508_18468_b200 as P  # noqa: E402
tr = P.Trajectories(16384, 1, "projective_events", [0.3], seed=0, orthonormalizer="lowrank")
tr.step(2)
torch.cuda.synchronize()
print("events in last window:", tr.last_clicks(0))
