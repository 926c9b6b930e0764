"""Pins for oracle/philox.py: published known-answer vectors, the 53-bit mapping, statistics."""
import numpy as np

from conftest import golden
from oracle.philox import philox4x32_10, site_uniforms, gaussian_from_uniforms


def test_known_answer_vectors():
    rows = [l.split() for l in open(golden("philox4x32_10_kat.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        out = philox4x32_10(np.array([v[:4]], dtype=np.uint64), v[4:6])[0]
        assert [int(x) for x in out] == v[6:10]


def test_vectorised_equals_scalar():
    ctr = np.array([[i, 7, 3, 0] for i in range(17)], dtype=np.uint64)
    allx = philox4x32_10(ctr, (11, 0))
    for i in range(17):
        one = philox4x32_10(ctr[i:i + 1], (11, 0))[0]
        assert np.array_equal(one, allx[i])


def test_uniform_mapping_exact():
    """u0 = ((x0>>5)*2^26 + (x1>>6)) * 2^-53 is an exact 53-bit dyadic in [0,1)."""
    u0, u1 = site_uniforms(4096, 5, 2, 0x123456789)
    for u in (u0, u1):
        assert u.min() >= 0.0 and u.max() < 1.0
        k = u * 2.0 ** 53
        assert np.all(k == np.floor(k))
    ctr = np.zeros((1, 4), dtype=np.uint64)
    ctr[0] = [3, 5, 2, 0]
    x = philox4x32_10(ctr, (0x23456789, 0x1))[0]
    want = ((int(x[0]) >> 5) * 2 ** 26 + (int(x[1]) >> 6)) / 2.0 ** 53
    assert u0[3] == want


def test_counter_words_are_distinct_streams():
    a = site_uniforms(64, 0, 0, 0)[0]
    b = site_uniforms(64, 1, 0, 0)[0]
    c = site_uniforms(64, 0, 1, 0)[0]
    d = site_uniforms(64, 0, 0, 1)[0]
    assert not np.array_equal(a, b) and not np.array_equal(a, c) and not np.array_equal(a, d)


def test_gaussian_statistics():
    """Box-Muller output: mean 0, variance 1 over 1e6 draws (SPEC S:301 noise-variance idea)."""
    zs = []
    for s in range(16):
        u0, u1 = site_uniforms(65536, s, 0, 42)
        zs.append(gaussian_from_uniforms(u0, u1))
    z = np.concatenate(zs)
    assert z.size > 1_000_000
    assert abs(z.mean()) < 5 / np.sqrt(z.size)
    assert abs(z.var() - 1.0) < 0.01
    # fourth moment 3 (Gaussian), a check that cos/log pairing is right
    assert abs(np.mean(z ** 4) - 3.0) < 0.05
