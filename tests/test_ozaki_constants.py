"""The modular scheme's host constants (csrc/ozaki.cu through traj_ozaki_constants / traj_ozaki_roots; no
GPU): the moduli are odd, pairwise coprime, fit int8 residues and each has a square root j of -1 (so that
z -> (re + j im, re - j im) turns a complex product mod m into two real ones); beta keeps twice every
product below M/2 by Cauchy-Schwarz; and the kernel's arithmetic -- the plane map of the splits, the two
residue products, 2 Re = P+ + P- left unreduced and 2 Im = -j (P+ - P-), one Garner step per modulus pair
with a single modulo and a canonicalising subtraction, the fractional CRT on a 2^-36 grid in FP64 --
returns random Gaussian-integer products exactly to FP64 rounding, conjugated operands by the plane swap,
and a zero product as exactly 0 (emulated here with exact Python integers and the same FP64 operations)."""
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


def roots(lib, s):
    j = (ctypes.c_int32 * s)()
    assert lib.traj_ozaki_roots(s, j) == 0
    return list(j)


def test_rejects_unsupported(lib):
    m = (ctypes.c_int32 * 32)()
    b = ctypes.c_int32()
    d = (ctypes.c_double * 16)()
    M = ctypes.c_double()
    for s in (0, 3, 5, 17, 20):
        assert lib.traj_ozaki_constants(s, m, ctypes.byref(b), d, d, ctypes.byref(M)) == 1
        assert lib.traj_ozaki_roots(s, m) == 1


@pytest.mark.parametrize("s", [4, 8, 10, 16, 18])
def test_moduli_and_bit_budget(lib, s):
    m, beta, ch, cl, Md = consts(lib, s)
    j = roots(lib, s)
    assert all(2 <= x <= 256 and x % 2 == 1 for x in m)
    for i in range(s):
        assert (j[i] * j[i] + 1) % m[i] == 0 and 0 < j[i] < m[i]      # j^2 = -1 (mod m)
        for k in range(i):
            assert math.gcd(m[i], m[k]) == 1
    M = math.prod(m)
    assert abs(Md - M) <= M * 2.0 ** -52
    # |X| <= ||a||_2 ||b||_2 with each side < 2^beta (+0.5 sqrt(K) of rounding, K < 2^17); the combine
    # reconstructs 2X: 2X < M / 2.  The operands' 21-bit digit split needs |x| < 2^62.
    K = 2 ** 17
    assert 2 * (2 ** beta + 0.5 * math.sqrt(K)) ** 2 < M // 2
    assert beta <= 61
    assert beta == {4: 14, 8: 29, 10: 37, 16: 57, 18: 61}[s]
    for p in range(s // 2):
        mu = m[2 * p] * m[2 * p + 1]
        assert mu < 2 ** 16
        assert 2 * m[2 * p] < 4 * m[2 * p + 1] and m[2 * p] > m[2 * p + 1]   # the Garner step's unreduced inputs
        n = ch[p] * 2.0 ** 36
        assert n == int(n) and 0 <= n <= 2 ** 36            # ch on the 2^-36 grid: r ch exact for r < 2^16
        inv = pow(M // mu % mu, -1, mu)
        assert abs((ch[p] + cl[p]) - inv / mu) < 2.0 ** -80 + abs(cl[p]) * 2.0 ** -52


def _fma(a, b, c):
    """a b + c rounded once to FP64 (CUDA's fma)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _planes(re, im, m, j):
    """The splits' plane map for one Gaussian integer and one modulus: the stored int8 residues of
    z+ = re + j im and z- = re - j im (oz_split_*_kernel / plane_words)."""
    xr, ji = re % m, (im % m) * j % m
    return ((xr + ji + 128) % m) - 128, ((xr + m - ji + 128) % m) - 128


def _combine(Pp, Pm, m, j, ch, cl, Md):
    """The kernel's arithmetic (oz_combine_kernel / CrtPair) for one output element from the exact
    integer sums P+ = sum a+ b+ and P- = sum a- b- PER MODULUS (lists): returns (2 Re, 2 Im)."""
    sr = si = lr = li = 0.0
    for p in range(len(m) // 2):
        ma, mb = m[2 * p], m[2 * p + 1]
        inv = pow(ma % mb, -1, mb)
        ap, am = Pp[2 * p] % ma, Pm[2 * p] % ma            # the INT8 launch's epilogue: bytes in [0, m)
        bp, bm = Pp[2 * p + 1] % mb, Pm[2 * p + 1] % mb
        rea, ima = ap + am, ((ap + ma - am) * (ma - j[2 * p])) % ma
        reb, imb = bp + bm, ((bp + mb - bm) * (mb - j[2 * p + 1])) % mb
        mu = ma * mb
        rr = rea + ma * (((reb + 4 * mb - rea) * inv) % mb)
        ri = ima + ma * (((imb + 4 * mb - ima) * inv) % mb)
        assert reb + 4 * mb - rea >= 0 and imb + 4 * mb - ima >= 0
        assert 0 <= rr < 2 * mu and 0 <= ri < 2 * mu        # one canonicalising step suffices
        rr, ri = (rr - mu if rr >= mu else rr), (ri - mu if ri >= mu else ri)
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


def _product(A, B, m, j, ch, cl, Md, conj_a=False, conj_b=False):
    """One output element sum_k A_k B_k of Gaussian integers (lists of (re, im)) through the scheme:
    plane residues, exact integer sums of residue products, combine.  A conjugated operand swaps planes."""
    Pp, Pm = [], []
    for q in range(len(m)):
        pa = [_planes(re, im, m[q], j[q]) for re, im in A]
        pb = [_planes(re, im, m[q], j[q]) for re, im in B]
        ia, ib = (1, 0) if conj_a else (0, 1), (1, 0) if conj_b else (0, 1)
        assert all(-128 <= v <= 127 for t in pa + pb for v in t)
        Pp.append(sum(x[ia[0]] * y[ib[0]] for x, y in zip(pa, pb)))
        Pm.append(sum(x[ia[1]] * y[ib[1]] for x, y in zip(pa, pb)))
    return _combine(Pp, Pm, m, j, ch, cl, Md)


@pytest.mark.parametrize("s", [8, 16, 18])
def test_reconstruction_is_exact(lib, s):
    m, beta, ch, cl, Md = consts(lib, s)
    j = roots(lib, s)
    M = math.prod(m)
    rng = random.Random(s)
    K = 6
    lim = int(2 ** beta / math.sqrt(K) / 2)   # entries: |re| + |im| over K terms has 2-norm < 2^beta
    for it in range(300):
        # mixed magnitudes, signs and zeros
        def ent():
            e = rng.choice([lim, lim >> 7, lim >> 23, 3, 1])
            return rng.randrange(-e, e + 1), rng.randrange(-e, e + 1)
        A = [ent() for _ in range(K)]
        B = [ent() for _ in range(K)]
        for ca, cb in ((False, False), (True, False), (False, True)):
            wr = wi = 0
            for (ar, ai), (br, bi) in zip(A, B):
                ai2, bi2 = (-ai if ca else ai), (-bi if cb else bi)
                wr += ar * br - ai2 * bi2
                wi += ar * bi2 + ai2 * br
            assert abs(2 * wr) < M // 2 and abs(2 * wi) < M // 2
            gr, gi = _product(A, B, m, j, ch, cl, Md, ca, cb)
            # absolute error far below the operands' own rounding (~2^beta in these units), relative ~ FP64
            for got, want in ((gr, 2 * wr), (gi, 2 * wi)):
                assert abs(got - want) <= 2.0 ** -50 * abs(want) + 2.0 ** (math.log2(M) - 68), (it, ca, cb)


@pytest.mark.parametrize("s", [8, 16, 18])
def test_zero_product_is_exactly_zero(lib, s):
    m, beta, ch, cl, Md = consts(lib, s)
    j = roots(lib, s)
    assert _combine([0] * s, [0] * s, m, j, ch, cl, Md) == (0.0, 0.0)
    # orthogonal non-zero operands: (1 + i)(1) + (1)(-(1 + i)) = 0
    assert _product([(1, 1), (1, 0)], [(1, 0), (-1, -1)], m, j, ch, cl, Md) == (0.0, 0.0)
