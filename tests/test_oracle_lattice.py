"""Pins for oracle/lattice.py: worked examples, library expm, Bessel closed form, free-evolution closed forms."""
import numpy as np
import scipy.linalg
import scipy.special

from conftest import read_kv
from oracle import gaussian, lattice

EX = read_kv("spec_examples.txt")


def test_ring4_hopping_and_spectrum():
    H = lattice.hopping_matrix(4)
    assert list(H[0]) == EX["ring4_hopping_row0"]
    assert np.allclose(np.sort(np.linalg.eigvalsh(H)), EX["ring4_eigenvalues"], atol=1e-14)


def test_torus_neighbours_row_major():
    H = lattice.hopping_matrix(4, 4)
    assert list(np.nonzero(H[0])[0]) == [int(x) for x in EX["torus4x4_site0_neighbours"]]
    assert np.array_equal(H, H.T)
    assert np.allclose(H.sum(axis=1), 4.0)          # 4 neighbours, J = 1


def test_propagator_matches_expm_and_is_unitary():
    for (Lx, Ly) in [(8, 1), (10, 1), (4, 6), (5, 3)]:
        H = lattice.hopping_matrix(Lx, Ly, 1.0)
        K = lattice.propagator(H, 0.05)
        # the textbook eigendecomposition definition agrees to its own accuracy (~L eps)
        assert np.abs(K - lattice.propagator_eigh(H, 0.05)).max() < 1e-13
        assert np.abs(K @ K.conj().T - np.eye(Lx * Ly)).max() < 1e-14


def test_lattice_propagator_forms_agree():
    K1 = lattice.propagator(lattice.hopping_matrix(64), 0.05)
    K2 = lattice.propagator_ring_fourier(64, 1.0, 0.05)
    assert np.abs(K1 - K2).max() < 1e-14
    K2d = lattice.propagator_lattice(6, 8, 1.0, 0.05)
    Kdirect = scipy.linalg.expm(-1j * 0.05 * lattice.hopping_matrix(6, 8))
    assert np.abs(K2d - Kdirect).max() < 1e-14


def test_propagator_bessel_closed_form():
    """K_{ij} = sum_{n = j-i mod L} (-i)^|n| J_|n|(2 J dt)   (generating function of J_n)."""
    for L, J, dt in [(16, 1.0, 0.05), (6, 1.0, 0.7), (32, 0.5, 1.3)]:
        K = lattice.propagator(lattice.hopping_matrix(L, 1, J), dt)
        row = np.zeros(L, dtype=complex)
        for n in range(-60, 61):
            row[n % L] += (-1j) ** abs(n) * scipy.special.jv(abs(n), 2 * J * dt)
        assert np.abs(K[0] - row).max() < 1e-14
        assert np.abs(K[3] - np.roll(row, 3)).max() < 1e-14


def _s_finite(L, t, J=1.0):
    m = np.arange(L)
    return np.mean(np.cos(4 * J * t * np.cos(2 * np.pi * m / L)))


def test_free_evolution_closed_form_1d():
    """gamma = 0, Neel: n_i(t) = 1/2 + (-1)^i/(2L) sum_m cos(4 J t cos(2 pi m / L))."""
    L, dt = 64, 0.05
    K = lattice.propagator(lattice.hopping_matrix(L), dt)
    U = lattice.initial_state(L)
    sign = (-1.0) ** np.arange(L)
    for s in range(1, 201):
        U = K @ U
        if s % 20 == 0:
            n = gaussian.occupations(U)
            want = 0.5 + 0.5 * sign * _s_finite(L, s * dt)
            assert np.abs(n - want).max() < 1e-13


def test_free_evolution_bessel_limit():
    """Large-L limit n_i = 1/2 + (-1)^i J0(4t)/2 (north star), valid while J_L(4t) ~ 0."""
    L, dt = 128, 0.05
    K = lattice.propagator_ring_fourier(L, 1.0, dt)
    U = lattice.initial_state(L)
    for s in range(100):
        U = K @ U
    n = gaussian.occupations(U)
    want = 0.5 + 0.5 * (-1.0) ** np.arange(L) * scipy.special.j0(4 * 100 * dt)
    assert np.abs(n - want).max() < 1e-12


def test_free_evolution_closed_form_2d():
    """Checkerboard on a torus: n = 1/2 + (-1)^(x+y)/2 s_Lx(t) s_Ly(t)."""
    Lx, Ly, dt = 8, 6, 0.05
    K = lattice.propagator_lattice(Lx, Ly, 1.0, dt)
    U = lattice.initial_state(Lx, Ly)
    ys, xs = np.divmod(np.arange(Lx * Ly), Lx)
    for s in range(1, 61):
        U = K @ U
    t = 60 * dt
    want = 0.5 + 0.5 * (-1.0) ** (xs + ys) * _s_finite(Lx, t) * _s_finite(Ly, t)
    assert np.abs(gaussian.occupations(U) - want).max() < 1e-13


def test_initial_states():
    U = lattice.initial_state(8)
    assert np.array_equal(gaussian.occupations(U), [1, 0, 1, 0, 1, 0, 1, 0])
    U2 = lattice.initial_state(4, 4)
    ys, xs = np.divmod(np.arange(16), 4)
    assert np.array_equal(gaussian.occupations(U2), ((xs + ys) % 2 == 0).astype(float))
    assert U2.shape == (16, 8)
