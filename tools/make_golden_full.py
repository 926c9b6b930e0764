"""Write the full-size oracle fixtures for configs c3 and c5 (tests/golden/*_full.npz).

Imports only ``oracle/`` and ``workloads`` (seeded configuration records): every stored value is
computed by the CPU oracle, never by the CUDA path.  SURVEY §8(c) "GPU vs oracle, short runs":
"At c3 and c5, compare rows of C in blocks of 256 plus all S values".

Stored per config, for trajectory 0, seed 0, after ``steps`` projective steps of the config:

- ``clicks_<s>`` / ``occ_<s>``   the clicked sites of step s (ascending) and their outcomes
  (readings Q10, Q13, Q16);
- ``n``                          every occupation n_i = C_ii of the final state;
- ``rows<b>``                    4 row blocks [r0, r0 + 256) of C = U U^dag -- a window of
  ``W`` columns around the diagonal (``cols<b>``: W window columns + 32 random columns) and the
  sketch C[rows, :] @ Omega with Omega = ``omega`` (L x 8, +-1 entries), which sees every column;
- ``S``                          S_A for the config's regions (c3: A = [0, l),
  l = L/8, L/4, 3L/8, L/2, reading Q22; c5: the half system x < 80, reading Q23), and for c5 also
  S of the two strips, S of their union and I_2.

Run on the CPU host (8 cores: c3 about 10 minutes, c5 about 40):
    python tools/make_golden_full.py c3 [c5]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import workloads  # noqa: E402
from oracle import gaussian, lattice, protocols  # noqa: E402

W = 64            # diagonal-window columns per row block
NRAND = 32        # random columns per row block
BLOCK = 256       # rows per block
NPROBE = 8        # sketch width


def row_blocks(L: int):
    return [0, L // 4 + 37, L // 2 - 128, L - BLOCK]


def generate(name: str, steps: int):
    w = workloads.CONFIGS[name]()
    t0 = time.time()
    K = lattice.propagator_lattice(w.Lx, w.Ly, w.J, w.dt)
    U = lattice.initial_state(w.Lx, w.Ly)
    g = w.gammas[0]
    out = {}
    for s in range(steps):
        U, S, occ = protocols.projective_step(U, K, g, w.dt, s, 0, w.seed, form="block")
        out[f"clicks_{s}"] = S.astype(np.int64)
        out[f"occ_{s}"] = occ.astype(np.int8)
        print(f"{name} step {s}: {S.size} clicks, {int(occ.sum())} occupied, {time.time() - t0:.0f} s",
              flush=True)
    del K
    L = w.L
    out["n"] = gaussian.occupations(U)
    rng = np.random.Generator(np.random.PCG64(2508))
    omega = rng.choice(np.array([-1.0, 1.0]), size=(L, NPROBE))
    out["omega"] = omega.astype(np.int8)
    for b, r0 in enumerate(row_blocks(L)):
        rows = np.arange(r0, r0 + BLOCK)
        c0 = min(max(r0 + BLOCK // 2 - W // 2, 0), L - W)
        cols = np.concatenate([np.arange(c0, c0 + W),
                               np.sort(rng.choice(L, size=NRAND, replace=False))])
        Cb = U[rows] @ U.conj().T
        out[f"rows{b}"] = rows.astype(np.int64)
        out[f"cols{b}"] = cols.astype(np.int64)
        out[f"C{b}"] = Cb[:, cols]
        out[f"sketch{b}"] = Cb @ omega
        del Cb
    S_names, S_vals = [], []
    if name == "c3":
        for ell in (L // 8, L // 4, 3 * L // 8, L // 2):
            S_names.append(f"l{ell}")
            S_vals.append(gaussian.entanglement_entropy(U, np.arange(ell)))
            print(f"{name} S(l={ell}) = {S_vals[-1]!r}, {time.time() - t0:.0f} s", flush=True)
    else:
        A, B = w.regions["mi"]
        for nm, reg in (("half", w.regions["half"]), ("A", A), ("B", B), ("AB", np.concatenate([A, B]))):
            S_names.append(nm)
            S_vals.append(gaussian.entanglement_entropy(U, reg))
            print(f"{name} S({nm}) = {S_vals[-1]!r}, {time.time() - t0:.0f} s", flush=True)
        S_names.append("I2")
        S_vals.append(S_vals[1] + S_vals[2] - S_vals[3])
    out["S"] = np.array(S_vals)
    meta = {"config": name, "steps": steps, "traj": 0, "seed": w.seed, "gamma": g, "dt": w.dt,
            "L": L, "Lx": w.Lx, "Ly": w.Ly, "S_names": S_names, "block": BLOCK, "window": W,
            "random_cols": NRAND, "probes": NPROBE, "oracle_seconds": round(time.time() - t0, 1),
            "generator": "tools/make_golden_full.py (oracle/ only)"}
    out["meta"] = np.array(json.dumps(meta))
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                        f"{name}_full.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB) in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    STEPS = {"c3": 2, "c5": 1}
    for nm in sys.argv[1:] or ["c3", "c5"]:
        generate(nm, STEPS[nm])
