"""Pins for oracle/gaussian.py: worked values, invariants, Fock-space Schmidt entropies."""
import numpy as np
import pytest

from conftest import read_kv
from fock import FockSector
from oracle import gaussian, lattice
from workloads import random_matrix

EX = read_kv("spec_examples.txt")


def rand_state(L, N, seed):
    return gaussian.orthonormalize(random_matrix(L, N, seed))


def test_entropy_worked_values():
    assert gaussian.entropy_from_eigenvalues([0.5]) == pytest.approx(EX["entropy_half"][0], abs=1e-15)
    assert gaussian.entropy_from_eigenvalues([0.0, 1.0, 1.0, 0.0]) == 0.0
    # two modes at lambda: closed form 2 * h(lambda)
    lam = 0.3
    h = -(lam * np.log(lam) + (1 - lam) * np.log(1 - lam))
    assert gaussian.entropy_from_eigenvalues([lam, lam]) == pytest.approx(2 * h, rel=1e-15)
    with pytest.raises(gaussian.SpectrumError):
        gaussian.entropy_from_eigenvalues([1.0 + 1e-6])
    with pytest.raises(gaussian.SpectrumError):
        gaussian.entropy_from_eigenvalues([-1e-6])


def test_product_state_zero_entropy():
    U = lattice.initial_state(16)
    for A in (np.arange(8), np.arange(3), [0, 5, 9]):
        assert gaussian.entanglement_entropy(U, A) == 0.0


def test_correlation_invariants():
    U = rand_state(12, 6, 1)
    C = gaussian.correlation(U)
    assert np.abs(C - C.conj().T).max() < 1e-14
    assert np.abs(C @ C - C).max() < 1e-13
    assert abs(np.trace(C).real - 6) < 1e-13
    assert np.abs(U.conj().T @ U - np.eye(6)).max() < 1e-14


def test_entropy_complement_symmetry_and_gram_form():
    U = rand_state(20, 10, 2)
    A = np.array([0, 1, 2, 5, 7, 11, 13])
    Abar = np.setdiff1d(np.arange(20), A)
    SA = gaussian.entanglement_entropy(U, A)
    assert SA == pytest.approx(gaussian.entanglement_entropy(U, Abar), abs=1e-12)
    UA = U[A]
    S_gram = gaussian.entropy_from_eigenvalues(np.linalg.eigvalsh(UA.conj().T @ UA))
    assert SA == pytest.approx(S_gram, abs=1e-12)


def test_mutual_information_identities():
    U = rand_state(20, 10, 3)
    A, B = np.arange(0, 5), np.arange(10, 15)
    assert gaussian.mutual_information(U, A, B) >= -1e-8
    Ac = np.setdiff1d(np.arange(20), A)
    assert gaussian.mutual_information(U, A, Ac) == pytest.approx(2 * gaussian.entanglement_entropy(U, A), abs=1e-12)
    with pytest.raises(ValueError):
        gaussian.mutual_information(U, A, np.arange(3, 8))


def test_orthonormalize_gauge_invariance():
    """Column scaling and a random right-mixing leave C unchanged (SPEC S:142-144 idea)."""
    U = rand_state(16, 8, 4)
    C = gaussian.correlation(U)
    M = random_matrix(8, 8, 5)
    for V in (2.0 * U, U @ M):
        assert np.abs(gaussian.correlation(gaussian.orthonormalize(V)) - C).max() < 1e-12


def test_correlation_vs_fock():
    """<c_i^dag c_j> from many-body amplitudes equals conj(U U^dag) (reading Q19)."""
    L, N = 8, 4
    U = rand_state(L, N, 6)
    F = FockSector(L, N)
    psi = F.slater(U)
    assert abs(np.linalg.norm(psi) - 1) < 1e-13
    assert np.abs(F.correlation(psi) - gaussian.correlation_paper(U)).max() < 1e-13


@pytest.mark.parametrize("A", [[0, 1, 2, 3], [0, 2, 4, 6], [1, 2, 5], [7]])
def test_entropy_vs_fock_schmidt(A):
    """Gaussian S_A equals the Fock Schmidt entropy (with fermionic reorder signs)."""
    L, N = 8, 4
    U = rand_state(L, N, 7)
    F = FockSector(L, N)
    assert gaussian.entanglement_entropy(U, A) == pytest.approx(F.entropy(F.slater(U), A), abs=1e-12)


def _fock_nn(F, psi):
    """Connected density-density correlator <n_i n_j> - <n_i><n_j> by brute force."""
    L = F.L
    n = F.occupations(psi)
    nn = np.zeros((L, L))
    for k, b in enumerate(F.states):
        occ = np.array([(b >> i) & 1 for i in range(L)], dtype=float)
        nn += abs(psi[k]) ** 2 * np.outer(occ, occ)
    return nn - np.outer(n, n)


def test_density_correlation_vs_fock():
    """Eq. (2): C_ij = -D_ij D_ji is the connected <n_i n_j> (Wick), checked on the many-body state."""
    L, N = 8, 4
    U = rand_state(L, N, 30)
    F = FockSector(L, N)
    nn = _fock_nn(F, F.slater(U))
    Cr = gaussian.density_correlation(U)
    for r in range(1, L):
        want = np.mean([nn[i, i + r] for i in range(L - r)])
        assert Cr[r] == pytest.approx(want, abs=1e-13)


def test_particle_covariance_vs_fock():
    """Eq. (5): G_AB = -Cov(N_A, N_B) on the many-body state."""
    L, N = 8, 4
    U = rand_state(L, N, 31)
    F = FockSector(L, N)
    nn = _fock_nn(F, F.slater(U))
    A, B = [0, 1, 5], [3, 6, 7]
    assert gaussian.particle_covariance(U, A, B) == pytest.approx(-nn[np.ix_(A, B)].sum(), abs=1e-13)
    assert gaussian.particle_covariance(U, A, B) >= 0.0


def test_density_correlation_product_state_and_sum_rule():
    """Neel product state: C(r) = 0.  Sum rule of a pure Gaussian state with N particles:
    sum_j |C_ij|^2 = n_i, so summing -C(r)(L-r) over r (both orders) gives N - sum n_i^2."""
    U = lattice.initial_state(16)
    assert np.all(gaussian.density_correlation(U)[1:] == 0.0)
    U = rand_state(20, 10, 32)
    Cr = gaussian.density_correlation(U)
    L = 20
    tot = -2 * sum(Cr[r] * (L - r) for r in range(1, L))
    n = gaussian.occupations(U)
    assert tot == pytest.approx(10 - np.sum(n ** 2), abs=1e-12)
