"""Fock-space brute force in the fixed-N sector (L <= 12): the independent pin of the oracle.

Test helper only.  Nothing here uses the Gaussian-state formalism; it works on
many-body amplitudes psi(b) over bitstrings b with N bits set.

Conventions
-----------
Basis state |b> = c^dag_{o_1} c^dag_{o_2} ... c^dag_{o_N} |vac>, o_1 < o_2 < ... (ascending).
For |psi> = prod_k [sum_j U_jk c_j^dag] |vac> the amplitude is
psi(b) = det U[o(b), :].
c_j acting on |b> gives the sign (-1)^{#occupied modes < j}; c_i^dag inserting i
gives (-1)^{#occupied modes < i} (counted after the removal).
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.linalg


class FockSector:
    def __init__(self, L: int, N: int):
        self.L, self.N = L, N
        self.states = [sum(1 << i for i in occ) for occ in itertools.combinations(range(L), N)]
        self.index = {b: k for k, b in enumerate(self.states)}
        self.dim = len(self.states)

    def occ(self, b: int):
        return [i for i in range(self.L) if (b >> i) & 1]

    # -- operators
    def hop(self, i: int, j: int, b: int):
        """c_i^dag c_j |b> = sign |b'>, or None."""
        if not (b >> j) & 1:
            return None
        sign = (-1) ** bin(b & ((1 << j) - 1)).count("1")
        b2 = b & ~(1 << j)
        if (b2 >> i) & 1:
            return None
        sign *= (-1) ** bin(b2 & ((1 << i) - 1)).count("1")
        return sign, b2 | (1 << i)

    def hamiltonian(self, Htilde: np.ndarray) -> np.ndarray:
        """Many-body H = sum_ij H~_ij c_i^dag c_j on the sector."""
        H = np.zeros((self.dim, self.dim), dtype=np.complex128)
        for k, b in enumerate(self.states):
            for i in range(self.L):
                for j in range(self.L):
                    if Htilde[i, j] == 0:
                        continue
                    r = self.hop(i, j, b)
                    if r is not None:
                        H[self.index[r[1]], k] += Htilde[i, j] * r[0]
        return H

    # -- states
    def slater(self, U: np.ndarray) -> np.ndarray:
        return np.array([np.linalg.det(U[self.occ(b), :]) for b in self.states])

    def correlation(self, psi: np.ndarray) -> np.ndarray:
        """<c_i^dag c_j>."""
        D = np.zeros((self.L, self.L), dtype=np.complex128)
        for k, b in enumerate(self.states):
            if psi[k] == 0:
                continue
            for i in range(self.L):
                for j in range(self.L):
                    r = self.hop(i, j, b)
                    if r is not None:
                        D[i, j] += np.conj(psi[self.index[r[1]]]) * r[0] * psi[k]
        return D

    def occupations(self, psi):
        n = np.zeros(self.L)
        for k, b in enumerate(self.states):
            for i in range(self.L):
                if (b >> i) & 1:
                    n[i] += abs(psi[k]) ** 2
        return n

    def project(self, psi, j: int, occupied: bool):
        """Projective measurement of n_j; returns (renormalised psi, probability)."""
        keep = np.array([((b >> j) & 1) == int(occupied) for b in self.states])
        out = np.where(keep, psi, 0.0)
        p = float(np.sum(np.abs(out) ** 2))
        return (out / np.sqrt(p) if p > 0 else out), p

    def weight(self, psi, a):
        """prod_i exp(a_i n_i) on psi, renormalised (homodyne diagonal factor)."""
        f = np.array([np.exp(sum(a[i] for i in self.occ(b))) for b in self.states])
        out = psi * f
        return out / np.linalg.norm(out)

    def entropy(self, psi, A) -> float:
        """Von Neumann entropy of region A via the Schmidt decomposition, with the
        fermionic reordering sign that moves the A modes to the front."""
        A = sorted(int(x) for x in A)
        Abar = [i for i in range(self.L) if i not in A]
        rows, cols = {}, {}
        M = {}
        for k, b in enumerate(self.states):
            sign = 1
            for i in Abar:
                if not (b >> i) & 1:
                    continue
                for j in A:
                    if j > i and (b >> j) & 1:
                        sign = -sign
            ka = tuple((b >> i) & 1 for i in A)
            kb = tuple((b >> i) & 1 for i in Abar)
            rows.setdefault(ka, len(rows))
            cols.setdefault(kb, len(cols))
            M[(rows[ka], cols[kb])] = sign * psi[k]
        mat = np.zeros((len(rows), len(cols)), dtype=np.complex128)
        for (r, c), v in M.items():
            mat[r, c] = v
        s = np.linalg.svd(mat, compute_uv=False) ** 2
        s = s[s > 1e-300]
        return float(-np.sum(s * np.log(s)))


def propagator(sector: FockSector, Htilde: np.ndarray, dt: float) -> np.ndarray:
    return scipy.linalg.expm(-1j * dt * sector.hamiltonian(Htilde))
