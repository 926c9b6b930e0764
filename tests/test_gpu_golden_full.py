"""Full-size GPU vs oracle parity at configs c3 and c5 (SURVEY §8(c) "GPU vs oracle, short runs":
"at c3 and c5, compare rows of C in blocks of 256 plus all S values").

The expected values are ``tests/golden/c3_full.npz`` / ``c5_full.npz``, written by
``tools/make_golden_full.py`` from the CPU oracle alone (same seed, same Philox counters, trajectory
0).  The GPU runs the config through the C-ABI in the launch configuration bench.py times (one
trajectory on one GPU, dense K, CholeskyQR2) and must match:

- every step: the click count and the number of "occupied" outcomes, and after the step n_j at each
  clicked site equal to its outcome (0 or 1) -- the outcomes site by site;
- the final n_i for all L sites, 1e-10;
- four row blocks of C = U U^dag (256 rows each): a window of columns around the diagonal plus
  random columns element by element (1e-10), and the sketch C[rows, :] @ Omega (Omega +-1, L x 8),
  which sees every column of the block (4 sqrt(L) 1e-10: a 1e-10 error anywhere in a row shows);
- S_A for the config's regions and (c5) I_2 of the strips, 1e-8.
"""
import json
import os

import numpy as np
import pytest

import workloads
from conftest import golden

pytestmark = pytest.mark.gpu

C_TOL = 1e-10
S_TOL = 1e-8


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2508_18468_b200 import build
    build.build()
    import paper_2508_18468_b200 as P
    P.load_library()
    return P


def regions(w, names):
    out = {}
    for nm in names:
        if w.name == "c3":
            out[nm] = np.arange(int(nm[1:]))
        elif nm == "half":
            out[nm] = w.regions["half"]
        elif nm in ("A", "B"):
            out[nm] = w.regions["mi"][0 if nm == "A" else 1]
        elif nm == "AB":
            out[nm] = np.concatenate(w.regions["mi"])
    return out


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_full_size_matches_oracle_golden(P, name):
    import torch
    path = golden(f"{name}_full.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path}: run tools/make_golden_full.py {name}")
    g = np.load(path)
    meta = json.loads(str(g["meta"]))
    w = workloads.CONFIGS[name]()
    assert (meta["L"], meta["seed"], meta["gamma"], meta["dt"]) == (w.L, w.seed, w.gammas[0], w.dt)
    tr = P.Trajectories(w.Lx, w.Ly, w.protocol, [w.gammas[0]], dt=w.dt, J=w.J, seed=w.seed, traj_base=0)
    for s in range(meta["steps"]):
        tr.step(1)
        clicks, occ = g[f"clicks_{s}"], g[f"occ_{s}"].astype(bool)
        assert tr.last_clicks(0) == (clicks.size, int(occ.sum())), s
        n = tr.occupations()[0].cpu().numpy()
        assert np.abs(n[clicks] - occ.astype(float)).max() < 1e-10, s
    assert not tr.failed(0)
    n = tr.occupations()[0].cpu().numpy()
    assert np.abs(n - g["n"]).max() < C_TOL
    omega = torch.from_numpy(g["omega"].astype(np.complex128)).cuda()
    for b in range(4):
        rows, cols = g[f"rows{b}"], g[f"cols{b}"]
        Cb = tr.correlation_rows(0, int(rows[0]), rows.size)
        got = Cb[:, torch.from_numpy(cols).cuda()].cpu().numpy()
        assert np.abs(got - g[f"C{b}"]).max() < C_TOL, b
        sk = (Cb @ omega).cpu().numpy()
        assert np.abs(sk - g[f"sketch{b}"]).max() < 4 * np.sqrt(w.L) * C_TOL, b
        del Cb
    S_want = dict(zip(meta["S_names"], g["S"]))
    reg = regions(w, [k for k in meta["S_names"] if k != "I2"])
    for nm, A in reg.items():
        assert abs(tr.entropy(A)[0] - S_want[nm]) < S_TOL, nm
    if "I2" in S_want:
        A, B = w.regions["mi"]
        assert abs(tr.mutual_info(A, B)[0] - S_want["I2"]) < S_TOL
    tr.close()
