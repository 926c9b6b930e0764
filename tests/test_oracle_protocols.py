"""Pins for oracle/protocols.py against a Fock-space brute force with shared randoms,
plus the closed-form and invariant checks of SURVEY §8(c)."""
import numpy as np
import pytest

from fock import FockSector, propagator as fock_propagator
from oracle import gaussian, lattice, protocols
from oracle.philox import site_uniforms, gaussian_from_uniforms
from oracle.trajectory import OracleTrajectory
from workloads import random_matrix


def rand_state(L, N, seed):
    return gaussian.orthonormalize(random_matrix(L, N, seed))


# ---------------------------------------------------------------- single measurements
@pytest.mark.parametrize("occupied", [True, False])
def test_single_site_update_vs_fock(occupied):
    L, N, j = 7, 3, 2
    U = rand_state(L, N, 10)
    F = FockSector(L, N)
    psi, p = F.project(F.slater(U), j, occupied)
    u1 = 0.0 if occupied else 0.999999
    U2, occ = protocols.measure_site_sequential(U, j, u1)
    assert occ == occupied
    assert np.abs(F.correlation(psi) - gaussian.correlation_paper(U2)).max() < 1e-12
    # Born probability: p_j = D_jj
    pj = gaussian.occupations(U)[j]
    assert p == pytest.approx(pj if occupied else 1 - pj, abs=1e-13)


@pytest.mark.parametrize("occupied", [True, False])
def test_paper_equations_A1_A2_vs_fock(occupied):
    """Eq. (A1) and the sign-corrected Eq. (A2) reproduce the projected Fock state (reading Q15)."""
    L, N, j = 8, 4, 5
    U = rand_state(L, N, 11)
    F = FockSector(L, N)
    psi, _ = F.project(F.slater(U), j, occupied)
    D2 = protocols.update_D_paper(gaussian.correlation_paper(U), j, occupied)
    assert np.abs(F.correlation(psi) - D2).max() < 1e-12


def test_printed_A2_sign_is_wrong():
    """The sign printed in Eq. (A2) does not give the projected state."""
    L, N, j = 8, 4, 5
    U = rand_state(L, N, 11)
    F = FockSector(L, N)
    psi, _ = F.project(F.slater(U), j, False)
    D = gaussian.correlation_paper(U)
    col, row = D[:, j].copy(), D[j, :].copy()
    Dm = D - np.outer(col, row) / (1 - D[j, j].real)
    Dm[j, :] = 0
    Dm[:, j] = 0
    assert np.abs(F.correlation(psi) - Dm).max() > 1e-3


def test_eigenstate_measurement_is_certain():
    """Measuring an occupied site of a product state returns 'occupied' whatever u1 (Q17 guard)."""
    U = lattice.initial_state(8)
    for u1 in (0.0, 0.5, 0.999999999):
        U2, occ = protocols.measure_site_sequential(U, 2, u1)
        assert occ
        assert np.abs(gaussian.correlation(U2) - gaussian.correlation(U)).max() < 1e-15
        U3, occ3 = protocols.measure_site_sequential(U, 3, u1)
        assert not occ3


def test_block_equals_sequential():
    """Sampling on D_SS with Eq. (A1)/(A2) + the null-space block update equals the
    sequential rank-1 form (same outcomes, same C)."""
    L, N = 40, 20
    K = lattice.propagator(lattice.hopping_matrix(L), 0.05)
    U0 = rand_state(L, N, 12)
    for step in range(6):
        Ua, Sa, oa = protocols.projective_step(U0, K, 4.0, 0.05, step, 3, 99, form="block")
        Ub, Sb, ob = protocols.projective_step(U0, K, 4.0, 0.05, step, 3, 99, form="sequential")
        assert np.array_equal(Sa, Sb) and np.array_equal(oa, ob)
        assert Sa.size > 0
        assert np.abs(gaussian.correlation(Ua) - gaussian.correlation(Ub)).max() < 1e-12
        U0 = Ua


def test_measure_every_site():
    """gamma dt = 1: every site is measured, exactly N occupied, C diagonal 0/1, S_A = 0."""
    L, N = 16, 8
    K = lattice.propagator(lattice.hopping_matrix(L), 0.05)
    U = rand_state(L, N, 13)
    U2, S, occ = protocols.projective_step(U, K, 20.0, 0.05, 0, 0, 5)
    assert S.size == L and occ.sum() == N
    C = gaussian.correlation(U2)
    assert np.abs(C - np.diag(np.diag(C))).max() < 1e-12
    assert np.abs(np.diag(C).real - occ).max() < 1e-12
    assert gaussian.entanglement_entropy(U2, np.arange(L // 2)) == pytest.approx(0.0, abs=1e-10)


def test_born_statistics():
    """Fixed state, one site: the occupied frequency is p within 4 sigma over 4000 Philox draws."""
    U = rand_state(10, 5, 14)
    p = gaussian.occupations(U)[4]
    hits = 0
    n = 4000
    for s in range(n):
        _, u1 = site_uniforms(10, s, 0, 77)
        hits += protocols.decide(p, u1[4])
    assert abs(hits / n - p) < 4 * np.sqrt(p * (1 - p) / n)


# ---------------------------------------------------------------- full trajectories vs Fock
def _fock_projective_run(L, gamma, dt, steps, seed, traj):
    N = L // 2
    H = lattice.hopping_matrix(L)
    F = FockSector(L, N)
    P = fock_propagator(F, H, dt)
    psi = F.slater(lattice.initial_state(L).astype(complex))
    out = []
    for s in range(steps):
        psi = P @ psi
        u0, u1 = site_uniforms(L, s, traj, seed)
        for j in np.nonzero(u0 < gamma * dt)[0]:
            p = F.occupations(psi)[j]
            occ = protocols.decide(float(p), float(u1[j]))
            psi, _ = F.project(psi, int(j), occ)
        out.append(F.correlation(psi))
    return out


def test_projective_trajectory_vs_fock():
    L, gamma, dt, steps = 8, 2.0, 0.05, 60
    ref = _fock_projective_run(L, gamma, dt, steps, seed=3, traj=1)
    tr = OracleTrajectory(L, 1, "projective", gamma, dt, seed=3, traj=1)
    clicks = 0
    for s in range(steps):
        tr.step()
        clicks += tr.last_clicks[0].size
        assert np.abs(np.conj(tr.correlation()) - ref[s]).max() < 1e-12
    assert clicks > 20


def test_homodyne_trajectory_vs_fock():
    """Split-step QSD (Eq. A3) is exact on the many-body state: the Fock state
    propagated by exp(-iH dt) then weighted by prod exp(a_i n_i) matches the oracle."""
    L, gamma, dt, steps = 8, 1.0, 0.05, 100
    N = L // 2
    F = FockSector(L, N)
    P = fock_propagator(F, lattice.hopping_matrix(L), dt)
    psi = F.slater(lattice.initial_state(L).astype(complex))
    tr = OracleTrajectory(L, 1, "homodyne", gamma, dt, seed=8, traj=2)
    for s in range(steps):
        psi = P @ psi
        n = F.occupations(psi)
        u0, u1 = site_uniforms(L, s, 2, 8)
        a = protocols.homodyne_factor(n, gaussian_from_uniforms(u0, u1), gamma, dt)
        psi = F.weight(psi, a)
        tr.step()
        assert np.abs(np.conj(tr.correlation()) - F.correlation(psi)).max() < 1e-12
    A = [0, 1, 2, 3]
    assert tr.entropy(A) == pytest.approx(F.entropy(psi, A), abs=1e-11)


def test_homodyne_special_cases():
    # J = 0: a product state is a fixed point, entropy stays exactly 0.
    tr = OracleTrajectory(12, 1, "homodyne", 1.0, 0.05, J=0.0, seed=1)
    C0 = tr.correlation()
    tr.step(20)
    assert np.abs(tr.correlation() - C0).max() < 1e-14
    assert tr.entropy(np.arange(6)) == 0.0
    # gamma = 0: reduces to free evolution (finite-L closed form)
    L, dt = 32, 0.05
    tr = OracleTrajectory(L, 1, "homodyne", 0.0, dt, seed=1)
    tr.step(40)
    m = np.arange(L)
    sfin = np.mean(np.cos(4 * 40 * dt * np.cos(2 * np.pi * m / L)))
    want = 0.5 + 0.5 * (-1.0) ** np.arange(L) * sfin
    assert np.abs(np.diag(tr.correlation()).real - want).max() < 1e-13


def test_homodyne_noise_variance():
    """dW_i = sqrt(gamma dt) z_i has variance gamma dt within 1% over 1e6 draws."""
    g, dt = 0.7, 0.05
    dw = []
    for s in range(16):
        u0, u1 = site_uniforms(65536, s, 0, 3)
        dw.append(protocols.homodyne_factor(np.full(65536, 0.5), gaussian_from_uniforms(u0, u1), g, dt))
    dw = np.concatenate(dw)
    assert abs(dw.var() / (g * dt) - 1) < 0.01


def test_zeno_pinning():
    """Very strong homodyne monitoring pins the state: S_A stays small (SPEC S:295 idea)."""
    tr = OracleTrajectory(24, 1, "homodyne", 200.0, 0.05, seed=4)
    tr.step(40)
    weak = OracleTrajectory(24, 1, "homodyne", 0.1, 0.05, seed=4)
    weak.step(40)
    assert tr.entropy(np.arange(12)) < 0.2 < weak.entropy(np.arange(12))


# ---------------------------------------------------------------- NEXT-2: RK4 QSD
def test_rk4_step_is_fourth_order_taylor_of_expm():
    """One RK4 step of the linear ODE dU/dt = M U equals exp(dt M) U up to the Taylor remainder
    |dt M|^5 / 5! (classical RK4 on a linear autonomous system), with M the Eq. (A3) generator."""
    import scipy.linalg
    L, gamma, dt = 12, 1.5, 0.05
    H = lattice.hopping_matrix(L)
    U = rand_state(L, 6, 40)
    n = gaussian.occupations(U)
    u0, u1 = site_uniforms(L, 3, 0, 1)
    dW = np.sqrt(gamma * dt) * gaussian_from_uniforms(u0, u1)
    M = protocols.qsd_generator(H, n, dW, gamma, dt)
    k1 = M @ U
    k2 = M @ (U + 0.5 * dt * k1)
    k3 = M @ (U + 0.5 * dt * k2)
    k4 = M @ (U + dt * k3)
    rk = U + dt / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    ex = scipy.linalg.expm(dt * M) @ U
    nrm = np.linalg.norm(dt * M, 2)
    bound = nrm ** 5 / 120 * np.exp(nrm) * np.linalg.norm(U, 2)
    assert np.linalg.norm(rk - ex, 2) <= bound
    # and the 4th-order Taylor polynomial is the same map (RK4 == Taylor-4 for linear M)
    X = dt * M
    tay = U + X @ U + X @ X @ U / 2 + X @ X @ X @ U / 6 + X @ X @ X @ X @ U / 24
    assert np.abs(rk - tay).max() < 1e-14


def test_rk4_free_evolution_converges_at_fourth_order():
    """gamma = 0: RK4 + QR against the finite-L closed form; halving dt cuts the error ~16x."""
    L, T = 32, 2.0
    m = np.arange(L)
    want = 0.5 + 0.5 * (-1.0) ** m * np.mean(np.cos(4 * T * np.cos(2 * np.pi * m / L)))
    errs = []
    for dt in (0.1, 0.05):
        tr = OracleTrajectory(L, 1, "homodyne_rk4", 0.0, dt, seed=0)
        tr.step(int(round(T / dt)))
        errs.append(np.abs(gaussian.occupations(tr.U) - want).max())
    assert errs[1] < 1e-5
    assert 10 < errs[0] / errs[1] < 24


def test_rk4_qsd_step_vs_fock_exponential():
    """Eq. (A3) on the many-body state: exp(sum_ij X_ij c_i^dag c_j)|psi> (X = dt M) is the Slater
    state of exp(X) U exactly; the RK4 step approximates it within the Taylor remainder
    |X|^5 e^|X| / 5! (the O(sqrt(dt)) noise term makes |X| ~ 0.5 at dt = 0.05)."""
    import scipy.linalg
    L, N, gamma, dt = 8, 4, 1.0, 0.05
    H = lattice.hopping_matrix(L)
    U = rand_state(L, N, 41)
    F = FockSector(L, N)
    n = gaussian.occupations(U)
    u0, u1 = site_uniforms(L, 0, 0, 9)
    dW = np.sqrt(gamma * dt) * gaussian_from_uniforms(u0, u1)
    X = dt * protocols.qsd_generator(H, n, dW, gamma, dt)
    psi = scipy.linalg.expm(F.hamiltonian(X)) @ F.slater(U)      # sum_ij X_ij c_i^dag c_j
    psi /= np.linalg.norm(psi)
    Ue = gaussian.orthonormalize(scipy.linalg.expm(X) @ U)
    assert np.abs(F.correlation(psi) - gaussian.correlation_paper(Ue)).max() < 1e-12
    U2 = protocols.homodyne_step_rk4(U, H, gamma, dt, 0, 0, 9)
    x = np.linalg.norm(X, 2)
    drift = np.linalg.norm(gaussian.correlation(U2) - gaussian.correlation(Ue), 2)
    assert drift < 4 * x ** 5 * np.exp(x) / 120 * np.linalg.cond(scipy.linalg.expm(X))


# ---------------------------------------------------------------- NEXT-4: event-driven PM
def test_event_pm_vs_fock():
    """The literal D-matrix PM against the Fock space with the same events:
    propagate by exp(-iH tau), project site j with Born p_j (the same p_c)."""
    from oracle.pm_events import EventPM
    from oracle.philox import event_uniforms
    L, gamma, dt = 8, 3.0, 0.05
    pm = EventPM(L, 1, gamma, dt, seed=4, traj=2)
    pm.step(40)
    assert len(pm.log) > 20
    F = FockSector(L, L // 2)
    H = lattice.hopping_matrix(L)
    import scipy.linalg
    Hm = F.hamiltonian(H)
    psi = F.slater(lattice.initial_state(L).astype(complex))
    t = 0.0
    for e, te, j, occ in pm.log:
        psi = scipy.linalg.expm(-1j * Hm * (te - t)) @ psi
        t = te
        _, u_site, u_pc = event_uniforms(e, 2, 4)
        assert j == int(u_site * L)
        p = F.occupations(psi)[j]
        assert protocols.decide(float(p), u_pc) == occ
        psi, _ = F.project(psi, j, occ)
    psi = scipy.linalg.expm(-1j * Hm * (40 * dt - t)) @ psi
    # C = U U^dag = conj(<c^dag c>) (reading Q19)
    assert np.abs(np.conj(F.correlation(psi)) - pm.correlation()).max() < 1e-11


def test_event_pm_rates_and_invariants():
    """Events arrive at rate gamma N, sites uniformly; D stays a rank-N projector."""
    from oracle.pm_events import EventPM
    L, gamma, dt = 40, 2.0, 0.05
    pm = EventPM(L, 1, gamma, dt, seed=1)
    pm.step(100)
    T = 100 * dt
    n_ev = len(pm.log)
    lam = gamma * (L // 2) * T
    assert abs(n_ev - lam) < 5 * np.sqrt(lam)
    C = pm.correlation()
    assert np.abs(C @ C - C).max() < 1e-10
    assert abs(np.trace(C).real - L // 2) < 1e-10
