import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2508_18468_b200 as P
L=256
for proto, gam in [("homodyne", 1.0), ("projective", 0.0), ("projective", 4.0)]:
    a = P.Trajectories(L, 1, proto, [gam], seed=13, shard_size=2)
    b = P.Trajectories(L, 1, proto, [gam], seed=13)
    for s in range(3):
        a.step(1); b.step(1)
        ca = a.correlation(0).cpu().numpy(); cb = b.correlation(0).cpu().numpy()
        print(proto, gam, s, "dC", np.abs(ca-cb).max(), "clicks", a.last_clicks(0), b.last_clicks(0),
              "n_a", a.occupations()[0].cpu().numpy()[:4], "n_b", b.occupations()[0].cpu().numpy()[:4])
