"""Pins of the Eq. (A3) drift term (2<n> - 1) gamma dt that do not re-use its formula.

Eq. (A3) is a quantum-state-diffusion unravelling of continuous monitoring of every n_i with
noise dW_i dW_j = delta_ij gamma dt.  Two properties of that unravelling are fixed by the
mathematics, independently of how the oracle writes the exponent:

1. **Born-rule martingale.**  With J = 0 the monitored observables commute with H, so the
   ensemble average of every occupation is conserved: E[n_i(t+dt)] = n_i(t).  A first-order
   (Euler / Lie) discretisation keeps it to O(dt^2) per step -- *only* with the drift 2<n>gamma dt;
   any other coefficient (n - 1, 1 - 2n, 4n - 1, none) leaves an O(dt) bias.
2. **Lindblad average.**  The average state obeys d rho/dt = gamma sum_i D[n_i] rho, so for
   i != j the averaged correlation decays as dE[C_ij]/dt = -gamma C_ij (n_i^2 = n_i).  This fixes
   the noise variance (gamma dt) and the drift jointly; the discrete one-step rate is
   -gamma + O(dt), and the Richardson extrapolation 2 r(dt/2) - r(dt) is -gamma + O(dt^2).

Expectations over the Gaussian noise are computed *exactly* (to quadrature precision) by a
tensor Gauss-Hermite rule over z: the oracle's own ``homodyne_step`` / ``homodyne_step_rk4``
run once per quadrature node, with the node fed in place of the Box-Muller draw (the Philox
stream itself is pinned separately by the Random123 known-answer vectors).  No statistics,
no tolerance on sampling noise.

``test_pins_reject_mutants`` runs the same checks on deliberately wrong drift / variance
coefficients and requires every mutant to fail at least one of them.
"""
import itertools

import numpy as np
import pytest

from oracle import gaussian, protocols

DTS = (0.05, 0.025, 0.0125)


def _state(L, N, seed):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((L, N)) + 1j * rng.standard_normal((L, N))
    return gaussian.orthonormalize(M)


def _expectations(monkeypatch, which, U, gamma, dt, order):
    """E[n'] and E[C'] after one J = 0 step, by tensor Gauss-Hermite quadrature over z."""
    L = U.shape[0]
    x, w = np.polynomial.hermite_e.hermegauss(order)     # weight exp(-z^2 / 2)
    w = w / np.sqrt(2.0 * np.pi)
    En = np.zeros(L)
    EC = np.zeros((L, L), dtype=np.complex128)
    for idx in itertools.product(range(order), repeat=L):
        z = x[list(idx)]
        wt = float(np.prod(w[list(idx)]))
        monkeypatch.setattr(protocols, "gaussian_from_uniforms", lambda u0, u1, z=z: z)
        if which == "split":
            U2 = protocols.homodyne_step(U, np.eye(L), gamma, dt, 0, 0, 0)
        else:
            U2 = protocols.homodyne_step_rk4(U, np.zeros((L, L)), gamma, dt, 0, 0, 0)
        C = gaussian.correlation(U2)
        En += wt * np.diag(C).real
        EC += wt * C
    return En, EC


def _martingale_bias(monkeypatch, which, U, gamma, order):
    n0 = gaussian.occupations(U)
    return [np.abs(_expectations(monkeypatch, which, U, gamma, dt, order)[0] - n0).max()
            for dt in DTS]


def _dephasing_rates(monkeypatch, which, U, gamma, order):
    """One-step rates r(dt) = (E[C'_ij] - C_ij) / (C_ij dt) for every i != j."""
    C0 = gaussian.correlation(U)
    off = ~np.eye(U.shape[0], dtype=bool)
    out = []
    for dt in DTS:
        EC = _expectations(monkeypatch, which, U, gamma, dt, order)[1]
        out.append(((EC - C0)[off] / (C0[off] * dt)))
    return out


def _martingale_ok(bias, gamma):
    # O((gamma dt)^2): below 0.6 (gamma dt)^2 at every dt and ~4x smaller when dt halves
    small = all(b <= 0.6 * (gamma * dt) ** 2 for b, dt in zip(bias, DTS))
    second_order = all(3.0 < bias[k] / bias[k + 1] < 5.0 for k in range(len(bias) - 1))
    return small and second_order


def _lindblad_ok(rates, gamma):
    # raw rate -gamma (1 + O(gamma dt)); Richardson 2 r(dt/2) - r(dt) = -gamma (1 + O((gamma dt)^2))
    gdt = gamma * DTS[-1]
    rich = [2 * rates[k + 1] - rates[k] for k in range(len(rates) - 1)]
    raw_ok = np.abs(rates[-1] + gamma).max() < 2.5 * gdt * gamma
    rich_ok = np.abs(rich[-1] + gamma).max() < 12.0 * gdt * gdt * gamma
    return bool(raw_ok and rich_ok)


CASES = [
    # (L, N, gamma, quadrature order, state)
    (2, 1, 1.0, 24, np.array([[np.sqrt(0.3)], [np.sqrt(0.7) * np.exp(0.4j)]])),
    (3, 1, 0.6, 14, None),
    (3, 2, 1.7, 14, None),
]


@pytest.mark.parametrize("which", ["split", "rk4"])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_born_rule_martingale(monkeypatch, which, case):
    L, N, gamma, order, U = CASES[case]
    U = _state(L, N, 30 + case) if U is None else U
    bias = _martingale_bias(monkeypatch, which, U, gamma, order)
    assert _martingale_ok(bias, gamma), bias


@pytest.mark.parametrize("which", ["split", "rk4"])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_lindblad_dephasing_rate(monkeypatch, which, case):
    L, N, gamma, order, U = CASES[case]
    U = _state(L, N, 30 + case) if U is None else U
    rates = _dephasing_rates(monkeypatch, which, U, gamma, order)
    assert _lindblad_ok(rates, gamma), [r.real for r in rates]


SPLIT_MUTANTS = {
    "(n-1)":   lambda n, z, g, dt: np.sqrt(g * dt) * z + (n - 1.0) * g * dt,
    "(1-2n)":  lambda n, z, g, dt: np.sqrt(g * dt) * z + (1.0 - 2.0 * n) * g * dt,
    "(4n-1)":  lambda n, z, g, dt: np.sqrt(g * dt) * z + (4.0 * n - 1.0) * g * dt,
    "no drift": lambda n, z, g, dt: np.sqrt(g * dt) * z,
    "var 2gdt": lambda n, z, g, dt: np.sqrt(2 * g * dt) * z + (2.0 * n - 1.0) * g * dt,
    "var gdt/2": lambda n, z, g, dt: np.sqrt(0.5 * g * dt) * z + (2.0 * n - 1.0) * g * dt,
}
RK4_MUTANTS = {
    "(n-1)":   lambda H, n, dW, g, dt: -1j * H + np.diag(dW / dt + g * (n - 1.0)),
    "(1-2n)":  lambda H, n, dW, g, dt: -1j * H + np.diag(dW / dt + g * (1.0 - 2.0 * n)),
    "no drift": lambda H, n, dW, g, dt: -1j * H + np.diag(dW / dt),
    "dW/2dt":  lambda H, n, dW, g, dt: -1j * H + np.diag(dW / (2 * dt) + g * (2.0 * n - 1.0)),
}


@pytest.mark.parametrize("which,name", [("split", k) for k in SPLIT_MUTANTS] +
                         [("rk4", k) for k in RK4_MUTANTS])
def test_pins_reject_mutants(monkeypatch, which, name):
    """Each wrong coefficient fails the martingale or the Lindblad pin (on the L = 2 case)."""
    if which == "split":
        monkeypatch.setattr(protocols, "homodyne_factor", SPLIT_MUTANTS[name])
    else:
        monkeypatch.setattr(protocols, "qsd_generator", RK4_MUTANTS[name])
    L, N, gamma, order, U = CASES[0]
    ok_m = _martingale_ok(_martingale_bias(monkeypatch, which, U, gamma, order), gamma)
    ok_l = _lindblad_ok(_dephasing_rates(monkeypatch, which, U, gamma, order), gamma)
    assert not (ok_m and ok_l)
