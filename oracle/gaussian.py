"""Gaussian-state observables and orthonormalisation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

State: |psi> = prod_k [sum_j U_jk c_j^dag] |vac>, U^dag U = 1.
Correlation matrix: D_ij = <c_i^dag c_j>; with the product form above
D = conj(U U^dag) (reading Q19); the paper and the north star also write
D = U U^dag.  Parity is taken on C := U U^dag; spectra and |C_ij|^2 are
identical for both readings.
"""
from __future__ import annotations

import numpy as np

SPECTRUM_TOL = 1e-8     # eigenvalues outside [-tol, 1+tol] are an error (reading Q21)


class SpectrumError(ValueError):
    pass


def correlation(U: np.ndarray) -> np.ndarray:
    """C = U U^dag (L x L), the correlation matrix of P:209."""
    return U @ U.conj().T


def correlation_paper(U: np.ndarray) -> np.ndarray:
    """D_ij = <c_i^dag c_j> = conj(U U^dag) for the product form of P:200-202."""
    return np.conj(U @ U.conj().T)


def orthonormalize(U: np.ndarray) -> np.ndarray:
    """Householder QR, keep Q ("we perform a QR decomposition on the matrix U").

    Raises if U is numerically rank deficient (the state collapsed)."""
    Q, R = np.linalg.qr(U, mode="reduced")
    d = np.abs(np.diag(R))
    if d.size and d.min() <= 1e-12 * max(d.max(), 1e-300):
        raise np.linalg.LinAlgError("rank-deficient orbital matrix")
    return Q


def entropy_from_eigenvalues(lam: np.ndarray) -> float:
    """S = -sum[lam ln lam + (1-lam) ln(1-lam)], 0 ln 0 = 0, lam clamped to [0,1]."""
    lam = np.asarray(lam, dtype=np.float64)
    if lam.size and (lam.min() < -SPECTRUM_TOL or lam.max() > 1.0 + SPECTRUM_TOL):
        raise SpectrumError(f"spectrum outside [0,1]: [{lam.min()}, {lam.max()}]")
    lam = np.clip(lam, 0.0, 1.0)
    s = 0.0
    for x in lam:
        if 0.0 < x < 1.0:
            s -= x * np.log(x) + (1.0 - x) * np.log(1.0 - x)
    return float(s)


def entanglement_entropy(U: np.ndarray, A) -> float:
    """S_A from the eigenvalues of C restricted to A."""
    A = np.asarray(A, dtype=np.int64)
    if A.size == 0:
        return 0.0
    UA = U[A, :]
    CA = UA @ UA.conj().T
    return entropy_from_eigenvalues(np.linalg.eigvalsh(CA))


def mutual_information(U: np.ndarray, A, B) -> float:
    """I_2 = S_A + S_B - S_{A u B}, A and B disjoint."""
    A = np.asarray(A, dtype=np.int64)
    B = np.asarray(B, dtype=np.int64)
    if np.intersect1d(A, B).size:
        raise ValueError("regions overlap")
    AB = np.concatenate([A, B])
    return entanglement_entropy(U, A) + entanglement_entropy(U, B) - entanglement_entropy(U, AB)


def occupations(U: np.ndarray) -> np.ndarray:
    """n_i = sum_k |U_ik|^2 (<n_i>_t = sum_j U_ij U_ij^*)."""
    return np.sum(np.abs(U) ** 2, axis=1)


def density_correlation(U: np.ndarray) -> np.ndarray:
    """C(r) of Eq. (2) for a 1d chain: C_ij = -D_ij D_ji = -|C_ij|^2 (i != j),
    averaged over the pairs with |i - j| = r (i < j: L - r pairs), r = 1..L-1.
    Returns an array of length L with entry 0 unused (NaN)."""
    C = correlation(U)
    L = C.shape[0]
    out = np.full(L, np.nan)
    w = np.abs(C) ** 2
    for r in range(1, L):
        out[r] = -np.mean(np.diagonal(w, offset=r))
    return out


def particle_covariance(U: np.ndarray, A, B) -> float:
    """G_AB of Eq. (5): -sum_{i in A, j in B} C_ij with C_ij = -|D_ij|^2,
    i.e. sum |(U U^dag)_ij|^2 over i in A, j in B (A, B disjoint)."""
    A = np.asarray(A, dtype=np.int64)
    B = np.asarray(B, dtype=np.int64)
    if np.intersect1d(A, B).size:
        raise ValueError("regions overlap")
    CAB = U[A] @ U[B].conj().T
    return float(np.sum(np.abs(CAB) ** 2))
