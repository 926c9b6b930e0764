"""One trajectory, step by step (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

The paper runs each trajectory from the Neel state until t >= L/2 and samples
observables from D = U U^dag; trajectory and time averages are
P:57.  Reading Q24: a sample at step s is taken on the state after s
steps (s = 0 is the initial state).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import gaussian, lattice, protocols

HOMODYNE = "homodyne"
HOMODYNE_RK4 = "homodyne_rk4"      # NEXT-2: the paper's RK4 integrator
PROJECTIVE = "projective"


@dataclass
class OracleTrajectory:
    Lx: int
    Ly: int = 1
    protocol: str = PROJECTIVE
    gamma: float = 0.5
    dt: float = 0.05
    J: float = 1.0
    seed: int = 0
    traj: int = 0                      # global trajectory id (Philox counter word 2)
    K: np.ndarray | None = None        # optional shared propagator
    U: np.ndarray = field(init=False)
    step_index: int = field(init=False, default=0)
    last_clicks: tuple = field(init=False, default=())

    def __post_init__(self):
        if self.protocol == HOMODYNE_RK4:
            self.H = lattice.hopping_matrix(self.Lx, self.Ly, self.J)
        elif self.K is None:
            self.K = lattice.propagator_lattice(self.Lx, self.Ly, self.J, self.dt)
        self.U = lattice.initial_state(self.Lx, self.Ly)

    @property
    def L(self) -> int:
        return self.Lx * self.Ly

    def step(self, n: int = 1, form: str = "block"):
        for _ in range(n):
            s = self.step_index
            if self.protocol == HOMODYNE:
                self.U = protocols.homodyne_step(self.U, self.K, self.gamma, self.dt, s, self.traj, self.seed)
            elif self.protocol == HOMODYNE_RK4:
                self.U = protocols.homodyne_step_rk4(self.U, self.H, self.gamma, self.dt, s, self.traj, self.seed)
            else:
                self.U, S, occ = protocols.projective_step(self.U, self.K, self.gamma, self.dt, s,
                                                           self.traj, self.seed, form=form)
                self.last_clicks = (S, occ)
            self.step_index += 1

    def correlation(self) -> np.ndarray:
        return gaussian.correlation(self.U)

    def entropy(self, A) -> float:
        return gaussian.entanglement_entropy(self.U, A)

    def mutual_info(self, A, B) -> float:
        return gaussian.mutual_information(self.U, A, B)
