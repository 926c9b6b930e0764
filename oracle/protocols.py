"""The two monitoring protocols, one time step each.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Step order (reading Q5, the north star's order): propagate U <- K U, read the
occupations of K U, draw the randoms of (trajectory, step, site), apply the
monitor, re-orthonormalise with Householder QR.

Homodyne / QSD (Eq. A3):
    U(t+dt) ~ exp(-i H~ dt + dW + (2<n> - 1) gamma dt) U(t)
in Lie-split form (reading Q5): K first, then the diagonal factor
    a_i = dW_i + (2 n_i - 1) gamma dt,   dW_i = sqrt(gamma dt) z_i,  z_i ~ N(0,1)
(reading Q6: dW_i dW_j = delta_ij gamma dt; Q7: the "-1" kept literally).

Projective / PM (Eq. A1, A2): reading Q10, every site clicks with
probability gamma dt per step (u0_i < gamma dt); the clicked set S is visited in
ascending order (Q16); the outcome at site j is "occupied" iff u1_j < p_j, p_j the
Born probability conditioned on the earlier outcomes of the same step (P:174,
Q13); a drawn branch of probability < 1e-12 is replaced by the certain one (Q17).
Eq. (A2) is used with the corrected sign (+), reading Q15.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

from . import gaussian
from .philox import site_uniforms, gaussian_from_uniforms

IMPOSSIBLE = 1e-12     # reading Q17


# ----------------------------------------------------------------------------- homodyne
def homodyne_factor(n, z, gamma: float, dt: float):
    """a_i = sqrt(gamma dt) z_i + (2 n_i - 1) gamma dt  (Eq. A3 diagonal part)."""
    return np.sqrt(gamma * dt) * z + (2.0 * n - 1.0) * gamma * dt


def homodyne_step(U, K, gamma: float, dt: float, step: int, traj: int, seed: int):
    """One QSD step (Eq. A3, split form), then QR."""
    U = K @ U
    n = gaussian.occupations(U)
    u0, u1 = site_uniforms(U.shape[0], step, traj, seed)
    a = homodyne_factor(n, gaussian_from_uniforms(u0, u1), gamma, dt)
    U = np.exp(a)[:, None] * U
    return gaussian.orthonormalize(U)


# ----------------------------------------------------------------------------- projective
def decide(p: float, u1: float) -> bool:
    """Born rule with reading Q13 (occupied iff u1 < p) and the Q17 guard."""
    p = min(max(p, 0.0), 1.0)
    occ = u1 < p
    if occ and p < IMPOSSIBLE:
        occ = False
    elif (not occ) and (1.0 - p) < IMPOSSIBLE:
        occ = True
    return occ


def measure_site_sequential(U, j: int, u1: float):
    """Measure n_j on the orthonormal state U, U-form.

    occupied: new orbitals = e_j plus the part of span(U) with zero amplitude on j:
              w = conj(U_j.)/|U_j.|,  U <- U - (U w - e_j) w^dag   (stays orthonormal)
    empty:    every orbital projected by (1 - e_j e_j^dag), i.e. row j zeroed, then QR.
    Returns (U', occupied)."""
    p = float(np.sum(np.abs(U[j]) ** 2))
    occ = decide(p, u1)
    U = U.copy()
    if occ:
        w = U[j].conj() / np.linalg.norm(U[j])
        Uw = U @ w
        Uw[j] -= 1.0
        U -= np.outer(Uw, w.conj())
    else:
        U[j, :] = 0.0
        U = gaussian.orthonormalize(U)
    return U, occ


def update_D_paper(D, j: int, occupied: bool):
    """Eq. (A1) (occupied) or Eq. (A2) with the corrected sign (empty) on D_ii' = <c_i^dag c_i'>.

    A1: D_jj = 1; D_ji' = D_ij = 0 (i, i' != j); D_ii' - D_ji' D_ij / D_jj otherwise.
    A2: row/col j = 0;                           D_ii' + D_ji' D_ij / (1 - D_jj) otherwise
        (the paper prints "-", reading Q15)."""
    D = D.copy()
    col = D[:, j].copy()   # D_ij
    row = D[j, :].copy()   # D_ji'
    djj = D[j, j].real
    if occupied:
        D -= np.outer(col, row) / djj
        D[j, :] = 0.0
        D[:, j] = 0.0
        D[j, j] = 1.0
    else:
        D += np.outer(col, row) / (1.0 - djj)
        D[j, :] = 0.0
        D[:, j] = 0.0
    return D


def sample_outcomes_paper(D_SS, u1_S):
    """Sequential conditional Born sampling over S (ascending) on D restricted to S,
    with Eq. (A1)/(A2) as the conditioning step.  Returns a bool array (occupied)."""
    D = np.array(D_SS, dtype=np.complex128, copy=True)
    out = np.zeros(len(u1_S), dtype=bool)
    for t in range(len(u1_S)):
        occ = decide(float(D[t, t].real), float(u1_S[t]))
        out[t] = occ
        D = update_D_paper(D, t, occ)
    return out


def project_block(U, S1, S0):
    """State after P1(S1) P0(S0) on span(U): span(E_S1) + Z_S0 U X, X = null(U_S1) (SVD),
    Z_S0 zeroing rows S0; then Householder QR.  Equivalent to the sequential rank-1 form."""
    L, N = U.shape
    S1 = np.asarray(S1, dtype=np.int64)
    S0 = np.asarray(S0, dtype=np.int64)
    if S1.size:
        X = scipy.linalg.null_space(U[S1, :])
        V = U @ X
    else:
        V = U.copy()
    V[S0, :] = 0.0
    E = np.zeros((L, S1.size), dtype=np.complex128)
    E[S1, np.arange(S1.size)] = 1.0
    return gaussian.orthonormalize(np.concatenate([E, V], axis=1))


def projective_step(U, K, gamma: float, dt: float, step: int, traj: int, seed: int,
                    form: str = "block"):
    """One PM step.  Returns (U', S, occupied) with S the clicked sites (ascending)."""
    if gamma * dt > 1.0:
        raise ValueError("projective protocol needs gamma*dt <= 1")
    U = K @ U
    L = U.shape[0]
    u0, u1 = site_uniforms(L, step, traj, seed)
    S = np.nonzero(u0 < gamma * dt)[0]
    if form == "sequential":
        occ = np.zeros(S.size, dtype=bool)
        for t, j in enumerate(S):
            U, occ[t] = measure_site_sequential(U, int(j), float(u1[j]))
        U = gaussian.orthonormalize(U)
        return U, S, occ
    if S.size == 0:
        return gaussian.orthonormalize(U), S, np.zeros(0, dtype=bool)
    US = U[S, :]
    D_SS = np.conj(US @ US.conj().T)          # D = conj(U U^dag), reading Q19
    occ = sample_outcomes_paper(D_SS, u1[S])
    U = project_block(U, S[occ], S[~occ])
    return U, S, occ


# ----------------------------------------------------------------------------- NEXT-2: RK4 QSD
def qsd_generator(H, n, dW, gamma: float, dt: float):
    """M of Eq. (A3) divided by dt: dU/dt = M U with
    M = -i H~ + diag(dW/dt) + gamma diag(2 <n>_t - 1), held fixed over the step
    (dW and <n>_t taken at time t)."""
    return -1j * H + np.diag(dW / dt + gamma * (2.0 * n - 1.0))


def homodyne_step_rk4(U, H, gamma: float, dt: float, step: int, traj: int, seed: int):
    """Paper-literal QSD step: classical fourth-order Runge-Kutta on dU/dt = M U over dt
    with the Gaussian noise dW_i = sqrt(gamma dt) z_i held across the four stages, then QR."""
    n = gaussian.occupations(U)
    u0, u1 = site_uniforms(U.shape[0], step, traj, seed)
    dW = np.sqrt(gamma * dt) * gaussian_from_uniforms(u0, u1)
    M = qsd_generator(H, n, dW, gamma, dt)
    k1 = M @ U
    k2 = M @ (U + 0.5 * dt * k1)
    k3 = M @ (U + 0.5 * dt * k2)
    k4 = M @ (U + dt * k3)
    U = U + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    return gaussian.orthonormalize(U)
