"""Lattice, hopping matrix, propagator and initial state.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper: the 1d Hamiltonian H = J sum_i (c_i^dag c_{i+1} + h.c.) with periodic
boundary conditions, J = 1 ("The model"); its coefficient matrix
H~_ij = J delta_{i+-1,j} (App. A, below Eq. A3); the 2d model is "exactly
the same Hamiltonian ... defined on a square lattice".  Reading Q2:
2d site index = y*Lx + x (row-major), periodic in both directions.

Initial state (reading Q1): even sites (0-based) occupied in 1d, the
checkerboard (x+y even) in 2d; U0[:, k] = e_{site_k} with the occupied sites in
ascending order (the |psi> = prod_k sum_j U_jk c_j^dag form
is P:200-202).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg


def n_sites(Lx: int, Ly: int = 1) -> int:
    return Lx * Ly


def hopping_matrix(Lx: int, Ly: int = 1, J: float = 1.0) -> np.ndarray:
    """H~ (real symmetric, L x L): J on every periodic nearest-neighbour bond.

    Bonds are accumulated, so a 2-site ring gets 2J (the literal sum over i of
    c_i^dag c_{i+1} + h.c. visits the bond twice)."""
    L = Lx * Ly
    H = np.zeros((L, L))
    for y in range(Ly):
        for x in range(Lx):
            i = y * Lx + x
            nbrs = [y * Lx + (x + 1) % Lx]
            if Ly > 1:
                nbrs.append(((y + 1) % Ly) * Lx + x)
            for j in nbrs:
                if j == i:
                    continue
                H[i, j] += J
                H[j, i] += J
    return H


def propagator(H: np.ndarray, dt: float) -> np.ndarray:
    """K = exp(-i H~ dt) by scipy.linalg.expm (Pade scaling and squaring; a library
    primitive).  Reading Q4: exact K instead of the paper's RK4.

    (The eigendecomposition form V exp(-i eps dt) V^T, ``propagator_eigh``, is the
    textbook definition but LAPACK's eigenvectors of the degenerate ring spectrum are
    orthogonal only to ~L*eps, and that drift compounds over thousands of steps.)"""
    return scipy.linalg.expm(-1j * dt * np.asarray(H, dtype=np.float64))


def propagator_eigh(H: np.ndarray, dt: float) -> np.ndarray:
    """K = V diag(exp(-i eps dt)) V^T from H~ = V diag(eps) V^T (used as a cross-check)."""
    eps, V = scipy.linalg.eigh(H)
    return (V * np.exp(-1j * eps * dt)) @ V.T


def propagator_ring_fourier(L: int, J: float, dt: float) -> np.ndarray:
    """K for the 1d ring by its Fourier eigenbasis (H~ is circulant; eigenvalues 2J cos q).

    K_ij = (1/L) sum_q exp(-2 i J dt cos q) exp(i q (i - j)),  q = 2 pi m / L.
    Same operator as ``propagator(hopping_matrix(L), dt)`` for L >= 3; used for
    large L where a dense eigh is slow.  First row by FFT, then circulant fill."""
    q = 2.0 * np.pi * np.arange(L) / L
    lam = np.exp(-2j * J * dt * np.cos(q))
    # c_d = (1/L) sum_m lam_m exp(i q_m d)  (d = i - j)
    c = np.fft.ifft(lam)
    d = (np.arange(L)[:, None] - np.arange(L)[None, :]) % L
    return c[d]


def propagator_lattice(Lx: int, Ly: int, J: float, dt: float, dense_max: int = 1024) -> np.ndarray:
    """K on the lattice.  1d: expm of H~ (L <= dense_max) else the Fourier form.
    2d: K = K_y (x) K_x for row-major sites, since H~ = I (x) H~_x + H~_y (x) I with
    commuting terms."""
    if Ly == 1:
        if Lx <= dense_max:
            return propagator(hopping_matrix(Lx, 1, J), dt)
        return propagator_ring_fourier(Lx, J, dt)
    Kx = propagator_lattice(Lx, 1, J, dt, dense_max)
    Ky = propagator_lattice(Ly, 1, J, dt, dense_max)
    return np.kron(Ky, Kx)


def occupied_sites(Lx: int, Ly: int = 1) -> np.ndarray:
    """Neel / checkerboard occupied sites, ascending (readings Q1, Q2)."""
    if Ly == 1:
        return np.arange(0, Lx, 2)
    ys, xs = np.divmod(np.arange(Lx * Ly), Lx)
    return np.nonzero((xs + ys) % 2 == 0)[0]


def initial_state(Lx: int, Ly: int = 1) -> np.ndarray:
    """U0 (L x N, complex128): column k = e_{site_k} for the k-th occupied site."""
    L = Lx * Ly
    occ = occupied_sites(Lx, Ly)
    U = np.zeros((L, occ.size), dtype=np.complex128)
    U[occ, np.arange(occ.size)] = 1.0
    return U
