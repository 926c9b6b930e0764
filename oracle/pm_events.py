"""NEXT-4: the paper-literal event-driven projective protocol (App. A).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Exactly the algorithm of App. A on the L x L correlation matrix:
  * waiting times tau = -ln(eta) / (gamma N), eta uniform in (0, 1], N = L/2 (the
    printed ln(eta)/(gamma N) is negative, reading Q12);
  * between events D(t + tau) = e^{-iH tau} D(t) e^{iH tau}, written here for
    C := U U^dag (reading Q19: the orbitals evolve as U -> e^{-iH tau} U);
  * at an event a site j is chosen uniformly, p_j = C_jj, p_c uniform in [0, 1]:
    occupied iff p_j >= p_c (reading Q13/Q17 as for the discretised protocol);
  * Eq. (A1) (occupied) or the sign-corrected Eq. (A2) (empty), P:175-193 (reading Q15).
Random numbers of event e of trajectory tau come from philox.event_uniforms(e, tau, seed).
A "window" advances the time from s*dt to (s+1)*dt processing every event inside it.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

from . import lattice, protocols
from .philox import event_uniforms


class EventPM:
    def __init__(self, Lx: int, Ly: int = 1, gamma: float = 0.5, dt: float = 0.05, J: float = 1.0,
                 seed: int = 0, traj: int = 0):
        self.Lx, self.Ly, self.gamma, self.dt, self.seed, self.traj = Lx, Ly, gamma, dt, seed, traj
        self.L = Lx * Ly
        self.N = self.L // 2
        H = lattice.hopping_matrix(Lx, Ly, J)
        self.eps, self.V = scipy.linalg.eigh(H)
        U0 = lattice.initial_state(Lx, Ly)
        self.C = U0 @ U0.conj().T
        self.t = 0.0
        self.window = 0
        self.event = 0
        self.t_next = self._waiting_time(0)
        self.log = []          # (event, time, site, occupied)

    def _waiting_time(self, e: int) -> float:
        u_eta, _, _ = event_uniforms(e, self.traj, self.seed)
        return -np.log(1.0 - u_eta) / (self.gamma * self.N) if self.gamma > 0 else np.inf

    def _evolve(self, tau: float):
        if tau <= 0:
            return
        K = (self.V * np.exp(-1j * self.eps * tau)) @ self.V.T
        self.C = K @ self.C @ K.conj().T

    def step(self, n: int = 1):
        for _ in range(n):
            t_end = (self.window + 1) * self.dt
            while self.t_next < t_end:
                self._evolve(self.t_next - self.t)
                self.t = self.t_next
                _, u_site, u_pc = event_uniforms(self.event, self.traj, self.seed)
                j = min(int(u_site * self.L), self.L - 1)
                occ = protocols.decide(float(self.C[j, j].real), u_pc)
                self.C = protocols.update_D_paper(self.C, j, occ)
                self.log.append((self.event, self.t, j, occ))
                self.event += 1
                self.t_next = self.t + self._waiting_time(self.event)
            self._evolve(t_end - self.t)
            self.t = t_end
            self.window += 1

    def correlation(self) -> np.ndarray:
        return self.C

    def entropy(self, A) -> float:
        from . import gaussian
        A = np.asarray(A, dtype=np.int64)
        return gaussian.entropy_from_eigenvalues(np.linalg.eigvalsh(self.C[np.ix_(A, A)]))
