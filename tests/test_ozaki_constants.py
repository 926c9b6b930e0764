"""The modular scheme's host constants (csrc/ozaki.cu through traj_ozaki_constants; no GPU): the moduli are
pairwise coprime and fit int8 residues, beta keeps every product below M/2 by Cauchy-Schwarz, and the
kernel's reconstruction -- 3M residue sums left unreduced, one Garner step per modulus pair with a single
modulo and a canonicalising subtraction, the fractional CRT on a 2^-36 grid in FP64 -- returns random
integers anywhere in (-M/2, M/2) exactly to FP64 rounding, and a zero product as exactly 0 (emulated here
with exact Python integers and the same FP64 operations)."""
import ctypes
import math
import random
from fractions import Fraction

import numpy as np
import pytest


@pytest.fixture(scope="module")
def lib():
    from paper_2508_18468_b200 import binding
    return binding.load_library()


def consts(lib, s):
    m = (ctypes.c_int32 * s)()
    beta = ctypes.c_int32()
    ch = (ctypes.c_double * (s // 2))()
    cl = (ctypes.c_double * (s // 2))()
    M = ctypes.c_double()
    assert lib.traj_ozaki_constants(s, m, ctypes.byref(beta), ch, cl, ctypes.byref(M)) == 0
    return list(m), beta.value, list(ch), list(cl), M.value


def test_rejects_unsupported(lib):
    m = (ctypes.c_int32 * 16)()
    b = ctypes.c_int32()
    d = (ctypes.c_double * 8)()
    M = ctypes.c_double()
    for s in (0, 3, 5, 18):
        assert lib.traj_ozaki_constants(s, m, ctypes.byref(b), d, d, ctypes.byref(M)) == 1


@pytest.mark.parametrize("s", [4, 8, 10, 16])
def test_moduli_and_bit_budget(lib, s):
    m, beta, ch, cl, Md = consts(lib, s)
    assert all(2 <= x <= 256 for x in m)
    for i in range(s):
        for j in range(i):
            assert math.gcd(m[i], m[j]) == 1
    M = math.prod(m)
    assert abs(Md - M) <= M * 2.0 ** -52
    # |X| <= ||a||_2 ||b||_2 with each side < 2^beta (+0.5 sqrt(K) of rounding, K < 2^17): X < M / 2
    K = 2 ** 17
    assert (2 ** beta + 0.5 * math.sqrt(K)) ** 2 < M // 2
    assert beta == {4: 14, 8: 30, 10: 38, 16: 61}[s]
    for p in range(s // 2):
        mu = m[2 * p] * m[2 * p + 1]
        assert mu < 2 ** 16
        n = ch[p] * 2.0 ** 36
        assert n == int(n) and 0 <= n <= 2 ** 36            # ch on the 2^-36 grid: r ch exact for r < 2^16
        inv = pow(M // mu % mu, -1, mu)
        assert abs((ch[p] + cl[p]) - inv / mu) < 2.0 ** -80 + abs(cl[p]) * 2.0 ** -52


def _fma(a, b, c):
    """a b + c rounded once to FP64 (CUDA's fma)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _combine(P1, P2, P3, m, ch, cl, Md, neg2=False):
    """The kernel's arithmetic (oz_combine_kernel / CrtPair) for one output element."""
    sr = si = lr = li = 0.0
    for p in range(len(m) // 2):
        ma, mb = m[2 * p], m[2 * p + 1]
        inv = pow(ma % mb, -1, mb)
        a = [x % ma for x in (P1, P2, P3)]
        b = [x % mb for x in (P1, P2, P3)]
        if neg2:
            rea, ima = a[0] + a[1], a[2] + ma - a[0] + a[1]
            reb, imb = b[0] + b[1], b[2] + mb - b[0] + b[1]
        else:
            rea, ima = a[0] + ma - a[1], a[2] + 2 * ma - a[0] - a[1]
            reb, imb = b[0] + mb - b[1], b[2] + 2 * mb - b[0] - b[1]
        mu = ma * mb
        rr = rea + ma * (((reb + 4 * mb - rea) * inv) % mb)
        ri = ima + ma * (((imb + 4 * mb - ima) * inv) % mb)
        rr, ri = min(rr, rr - mu if rr >= mu else rr), min(ri, ri - mu if ri >= mu else ri)
        assert 0 <= rr < mu and 0 <= ri < mu
        n = int(ch[p] * 2.0 ** 36)
        assert rr * n < 2 ** 53 and ri * n < 2 ** 53          # r ch exact in FP64
        tr, ti = rr * ch[p], ri * ch[p]
        tr -= np.rint(tr)
        ti -= np.rint(ti)
        sr += tr
        si += ti
        lr = _fma(float(rr), cl[p], lr)
        li = _fma(float(ri), cl[p], li)

    def val(S, l):
        f = S - np.rint(S)
        f += l
        f -= np.rint(f)
        return f * Md
    return val(sr, lr), val(si, li)


@pytest.mark.parametrize("s", [8, 16])
def test_reconstruction_is_exact(lib, s):
    m, beta, ch, cl, Md = consts(lib, s)
    M = math.prod(m)
    rng = random.Random(s)
    lim = 2 ** (2 * beta)   # the products' range under the scaling
    for _ in range(3000):
        p1, p2, p3 = (rng.randrange(-lim, lim) for _ in range(3))
        re, im = p1 - p2, p3 - p1 - p2
        if abs(re) >= M // 2 or abs(im) >= M // 2:
            continue
        gr, gi = _combine(p1, p2, p3, m, ch, cl, Md)
        # absolute error far below the operands' own rounding (~2^beta in these units), relative ~ FP64
        for got, want in ((gr, re), (gi, im)):
            assert abs(got - want) <= 2.0 ** -50 * abs(want) + 2.0 ** (math.log2(M) - 68)
        # the conjugated Gram form: Re = P1 + P2', Im = P3 - P1 + P2'
        re2, im2 = p1 + p2, p3 - p1 + p2
        if abs(re2) < M // 2 and abs(im2) < M // 2:
            gr2, gi2 = _combine(p1, p2, p3, m, ch, cl, Md, neg2=True)
            for got, want in ((gr2, re2), (gi2, im2)):
                assert abs(got - want) <= 2.0 ** -50 * abs(want) + 2.0 ** (math.log2(M) - 68)


@pytest.mark.parametrize("s", [8, 16])
def test_zero_product_is_exactly_zero(lib, s):
    m, beta, ch, cl, Md = consts(lib, s)
    assert _combine(0, 0, 0, m, ch, cl, Md) == (0.0, 0.0)
    assert _combine(0, 0, 0, m, ch, cl, Md, neg2=True) == (0.0, 0.0)
