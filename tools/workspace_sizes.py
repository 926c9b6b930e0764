"""Per-handle workspace (device memory) of each config, as the library sizes it."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, workloads
import paper_2508_18468_b200 as P
for name, prop, tpg in [("c1", "dense", 16), ("c2", "dense", 8), ("c3", "dense", 1), ("c3", "banded", 1), ("c4", "dense", 8), ("c5", "dense", 1), ("c5", "banded", 1)]:
    w = workloads.CONFIGS[name]()
    g = [w.gammas[t % len(w.gammas)] for t in range(tpg)]
    tr = P.Trajectories(w.Lx, w.Ly, w.protocol, g, dt=w.dt, seed=0, propagator=prop)
    print(name, prop, tpg, "workspace GB", round(tr.workspace.numel() / 1e9, 2), flush=True)
    tr.close(); del tr; torch.cuda.empty_cache()
