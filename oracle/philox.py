"""Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as 1, 2, 3").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper does not say how its Gaussian noise or its measurement randoms are
drawn ("independent Gaussian random noise").  Reading
Q9: every random number of trajectory ``tau`` at step ``s`` on site
``i`` comes from one Philox4x32-10 block with

    counter = (i, s, tau_global, 0)      key = (seed & 0xffffffff, seed >> 32)

and two 53-bit uniforms in [0, 1):

    u0 = ((x0 >> 5) * 2**26 + (x1 >> 6)) * 2**-53
    u1 = ((x2 >> 5) * 2**26 + (x3 >> 6)) * 2**-53

Implemented here in NumPy uint64 arithmetic (multiply-high via 64-bit
products), vectorised over counters.  The CUDA side implements the same
generator independently with ``__umulhi``; the two never share code.
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def philox4x32_10(ctr, key):
    """Ten Philox4x32 rounds.

    ctr: uint array of shape (..., 4) with values < 2**32; key: two ints < 2**32.
    Returns uint64 array of shape (..., 4) holding the four 32-bit output words.
    """
    c = np.asarray(ctr, dtype=np.uint64) & _MASK
    c0, c1, c2, c3 = (c[..., j].copy() for j in range(4))
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + _W0) & 0xFFFFFFFF
            k1 = (k1 + _W1) & 0xFFFFFFFF
        p0 = _M0 * c0            # exact: both factors < 2**32
        p1 = _M1 * c2
        hi0, lo0 = p0 >> _S32, p0 & _MASK
        hi1, lo1 = p1 >> _S32, p1 & _MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0)
    return np.stack([c0, c1, c2, c3], axis=-1)


def _u53(a, b):
    return ((a >> np.uint64(5)).astype(np.float64) * 67108864.0
            + (b >> np.uint64(6)).astype(np.float64)) * (1.0 / 9007199254740992.0)


def site_uniforms(L: int, step: int, traj: int, seed: int):
    """(u0, u1) for sites 0..L-1 of trajectory ``traj`` at step ``step`` (Q9)."""
    ctr = np.zeros((L, 4), dtype=np.uint64)
    ctr[:, 0] = np.arange(L, dtype=np.uint64)
    ctr[:, 1] = np.uint64(step)
    ctr[:, 2] = np.uint64(traj)
    x = philox4x32_10(ctr, (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF))
    return _u53(x[:, 0], x[:, 1]), _u53(x[:, 2], x[:, 3])


def gaussian_from_uniforms(u0, u1):
    """Box-Muller (reading Q8): z = sqrt(-2 ln(1-u0)) cos(2 pi u1), one z per site."""
    return np.sqrt(-2.0 * np.log(1.0 - u0)) * np.cos(2.0 * np.pi * u1)


def event_uniforms(event: int, traj: int, seed: int):
    """The three uniforms of measurement event number `event` of the event-driven PM protocol
    (NEXT-4): counter (event_lo, event_hi, traj, 1) -> (u_eta, u_site),
    counter (event_lo, event_hi, traj, 2) -> u_pc (53-bit each, same mapping as site_uniforms)."""
    key = (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    c = np.array([[event & 0xFFFFFFFF, (event >> 32) & 0xFFFFFFFF, traj, 1],
                  [event & 0xFFFFFFFF, (event >> 32) & 0xFFFFFFFF, traj, 2]], dtype=np.uint64)
    x = philox4x32_10(c, key)
    return float(_u53(x[0:1, 0], x[0:1, 1])[0]), float(_u53(x[0:1, 2], x[0:1, 3])[0]), \
        float(_u53(x[1:2, 0], x[1:2, 1])[0])
