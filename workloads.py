"""Seeded synthetic workloads shared by the tests, bench.py and the oracle runs.

Holds NONE of the method's arithmetic: only configuration records (lattice,
protocol, gamma, dt, step counts, regions) taken from BASELINE.json ``configs``
and SURVEY.md §8(d), plus a seeded complex-Gaussian matrix generator for tests
that start from a random state.  The trajectory randoms themselves are drawn by
each side's own Philox4x32-10 (reading Q9), never passed through here.

The paper measures on no external dataset; every input is synthetic by
construction.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

HOMODYNE = "homodyne"
PROJECTIVE = "projective"


@dataclass(frozen=True)
class Workload:
    name: str
    Lx: int
    Ly: int
    protocol: str
    gammas: tuple
    dt: float = 0.05
    J: float = 1.0
    seed: int = 0
    n_traj_per_gamma: int = 1
    steps: int = 200
    sample_every: int = 10
    regions: dict = field(default_factory=dict)   # name -> site array (or (A, B) pair for MI)

    @property
    def L(self) -> int:
        return self.Lx * self.Ly

    @property
    def N(self) -> int:
        return self.L // 2

    @property
    def n_traj(self) -> int:
        return self.n_traj_per_gamma * len(self.gammas)

    def gamma_of(self, traj: int) -> float:
        """gamma-index folded into the global trajectory id."""
        return self.gammas[traj // self.n_traj_per_gamma]


def half_chain(L: int) -> np.ndarray:
    """A = [0, L/2) (reading Q22; P:49 uses the 1-based {1..L/2})."""
    return np.arange(L // 2)


def columns(Lx: int, Ly: int, x0: int, x1: int) -> np.ndarray:
    """All sites with x in [x0, x1), row-major site = y*Lx + x (reading Q23)."""
    ys, xs = np.divmod(np.arange(Lx * Ly), Lx)
    return np.nonzero((xs >= x0) & (xs < x1))[0]


def strips_2d(Lx: int, Ly: int):
    """A = x in [0, Lx/4), B = x in [Lx/2, 3Lx/4): L x L/4 blocks separated by an
    L x L/4 block (reading Q23)."""
    return columns(Lx, Ly, 0, Lx // 4), columns(Lx, Ly, Lx // 2, 3 * Lx // 4)


def c1() -> Workload:
    return Workload("c1", 64, 1, PROJECTIVE, (0.5,), n_traj_per_gamma=16, steps=200,
                    sample_every=10, regions={"half": half_chain(64)})


def c2() -> Workload:
    return Workload("c2", 2048, 1, HOMODYNE, (0.1, 0.3, 1.0), n_traj_per_gamma=64,
                    steps=20480, sample_every=20, regions={"half": half_chain(2048)})


def c3() -> Workload:
    L = 16384
    return Workload("c3", L, 1, PROJECTIVE, (0.3,), n_traj_per_gamma=1, steps=200,
                    sample_every=50,
                    regions={f"l{ell}": np.arange(ell) for ell in (L // 8, L // 4, 3 * L // 8, L // 2)})


def c4() -> Workload:
    return Workload("c4", 64, 64, HOMODYNE, tuple(np.linspace(0.5, 3.0, 8)), n_traj_per_gamma=32,
                    steps=1280, sample_every=20, regions={"mi": strips_2d(64, 64)})


def c5(stress: bool = False) -> Workload:
    # reading Q11: per-site gamma = 2.86 is the per-site equivalent of the paper's PM
    # gamma_c = 5.72; the stress variant takes 5.72 literally.
    g = 5.72 if stress else 2.86
    return Workload("c5", 160, 160, PROJECTIVE, (g,), n_traj_per_gamma=1, steps=100,
                    sample_every=20,
                    regions={"half": columns(160, 160, 0, 80), "mi": strips_2d(160, 160)})


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """Seeded complex Gaussian matrix (PCG64), e.g. a random full-rank orbital matrix."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((rows, cols)) + 1j * rng.standard_normal((rows, cols))
