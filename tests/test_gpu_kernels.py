"""Kernel-level checks of the building blocks through the C-ABI (traj_zgemm, traj_chol_inverse)
against plain NumPy on the same seeded inputs: all op combinations, ragged tails that span
several 128 x 64 tiles, batches, triangular skipping and the upper-only epilogue."""
import itertools

import numpy as np
import pytest

from workloads import random_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2508_18468_b200 import build
    build.build()
    import paper_2508_18468_b200 as P
    P.load_library()
    return torch


def dev(T, a):
    return T.from_numpy(np.ascontiguousarray(a)).cuda()


def opx(a, op):
    return a if op == 0 else a.conj().T


SHAPES = [(1, 1, 1), (7, 5, 3), (128, 64, 8), (130, 67, 19), (257, 190, 77), (64, 300, 1000), (33, 129, 520)]


@pytest.mark.parametrize("opA,opB", list(itertools.product((0, 1), (0, 1))))
def test_zgemm_ops_and_ragged_shapes(T, opA, opB):
    from paper_2508_18468_b200 import traj_zgemm
    for i, (M, N, K) in enumerate(SHAPES):
        A = random_matrix(*((M, K) if opA == 0 else (K, M)), seed=10 + i)
        B = random_matrix(*((K, N) if opB == 0 else (N, K)), seed=50 + i)
        ref = opx(A, opA) @ opx(B, opB)
        C = T.zeros((M, N), dtype=T.complex128, device="cuda")
        traj_zgemm(opA, opB, dev(T, A), dev(T, B), C, K=K)
        err = np.abs(C.cpu().numpy() - ref).max()
        assert err < 1e-13 * K * 8, (M, N, K, err)


def test_zgemm_alpha_beta_batch_shared_operand(T):
    from paper_2508_18468_b200 import traj_zgemm
    M, N, K, nb = 150, 90, 70, 3
    A = random_matrix(M, K, 1)
    Bs = np.stack([random_matrix(K, N, 2 + b) for b in range(nb)])
    C0 = np.stack([random_matrix(M, N, 9 + b) for b in range(nb)])
    C = dev(T, C0.copy())
    alpha = 0.3 - 1.7j
    traj_zgemm(0, 0, dev(T, A[None]), dev(T, Bs), C, alpha=alpha, beta=1.0)
    for b in range(nb):
        ref = alpha * A @ Bs[b] + C0[b]
        assert np.abs(C[b].cpu().numpy() - ref).max() < 1e-11


def test_zgemm_padded_leading_dimension(T):
    from paper_2508_18468_b200 import traj_zgemm
    M, N, K = 100, 50, 60
    Abig = dev(T, random_matrix(M, K + 8, 3))
    Bbig = dev(T, random_matrix(K, N + 16, 4))
    Cbig = T.zeros((M, N + 24), dtype=T.complex128, device="cuda")
    traj_zgemm(0, 0, Abig[:, :K], Bbig[:, :N], Cbig[:, :N], M=M, N=N, K=K)
    ref = Abig[:, :K].cpu().numpy() @ Bbig[:, :N].cpu().numpy()
    got = Cbig.cpu().numpy()
    assert np.abs(got[:, :N] - ref).max() < 1e-11
    assert np.all(got[:, N:] == 0)


def test_zgemm_triangular_skips_and_upper_epilogue(T):
    from paper_2508_18468_b200 import traj_zgemm, binding as b
    n, K = 300, 300
    X = np.triu(random_matrix(n, n, 5))
    A = random_matrix(K, n, 6)
    # B upper triangular: skip k > n0+BN
    C = T.zeros((K, n), dtype=T.complex128, device="cuda")
    traj_zgemm(0, 0, dev(T, A), dev(T, X), C, flags=b.TRAJ_TRI_B_UPPER)
    assert np.abs(C.cpu().numpy() - A @ X).max() < 1e-11
    # A upper triangular
    Bm = random_matrix(n, 77, 7)
    C = T.zeros((n, 77), dtype=T.complex128, device="cuda")
    traj_zgemm(0, 0, dev(T, X), dev(T, Bm), C, flags=b.TRAJ_TRI_A_UPPER)
    assert np.abs(C.cpu().numpy() - X @ Bm).max() < 1e-11
    # A lower (as op: X^dag is lower) and B lower
    C = T.zeros((n, 77), dtype=T.complex128, device="cuda")
    traj_zgemm(1, 0, dev(T, X), dev(T, Bm), C, flags=b.TRAJ_TRI_A_LOWER)
    assert np.abs(C.cpu().numpy() - X.conj().T @ Bm).max() < 1e-11
    C = T.zeros((K, n), dtype=T.complex128, device="cuda")
    traj_zgemm(0, 1, dev(T, A), dev(T, X), C, flags=b.TRAJ_TRI_B_LOWER)
    assert np.abs(C.cpu().numpy() - A @ X.conj().T).max() < 1e-11
    # Hermitian Gram, upper only: lower triangle untouched
    U = random_matrix(500, n, 8)
    G = T.full((n, n), 7.0 + 0j, dtype=T.complex128, device="cuda")
    traj_zgemm(1, 0, dev(T, U), dev(T, U), G, flags=b.TRAJ_C_UPPER)
    g = G.cpu().numpy()
    ref = U.conj().T @ U
    iu = np.triu_indices(n)
    il = np.tril_indices(n, -1)
    assert np.abs(g[iu] - ref[iu]).max() < 1e-10
    assert np.all(g[il] == 7.0)


@pytest.mark.parametrize("leaf", ["elim", "regs"])
@pytest.mark.parametrize("n", [1, 5, 17, 33, 64, 65, 130, 300, 520])
def test_chol_inverse(T, n, leaf, monkeypatch):
    """Both 64 x 64 leaves (the elimination leaf, default; TRAJ_CHOL_LEAF=regs the register-blocked
    one) under the recursion, against NumPy's Cholesky and inverse."""
    from paper_2508_18468_b200 import traj_chol_inverse
    monkeypatch.setenv("TRAJ_CHOL_LEAF", leaf)
    nb = 3
    Gs = []
    for b in range(nb):
        M = random_matrix(n + 7, n, 100 + b)
        Gs.append(M.conj().T @ M)
    Gs = np.stack(Gs)
    G = dev(T, Gs.copy())
    X = T.full((nb, n, n), 5.0 + 0j, dtype=T.complex128, device="cuda")
    X, failed = traj_chol_inverse(G, X)
    x = X.cpu().numpy()
    assert failed.cpu().numpy().sum() == 0
    for b in range(nb):
        R = np.linalg.cholesky(Gs[b]).conj().T        # G = R^dag R, R upper
        Xr = np.linalg.inv(R)
        assert np.all(x[b][np.tril_indices(n, -1)] == 0)
        assert np.abs(x[b] - Xr).max() / np.abs(Xr).max() < 1e-12
        assert np.abs(x[b].conj().T @ Gs[b] @ x[b] - np.eye(n)).max() < 1e-11


@pytest.mark.parametrize("leaf", ["elim", "regs"])
def test_chol_inverse_flags_breakdown(T, leaf, monkeypatch):
    from paper_2508_18468_b200 import traj_chol_inverse
    monkeypatch.setenv("TRAJ_CHOL_LEAF", leaf)
    n = 70
    M = random_matrix(n, n, 1)
    G = M.conj().T @ M
    G[40, 40] = -5.0
    X = T.zeros((n, n), dtype=T.complex128, device="cuda")
    _, failed = traj_chol_inverse(dev(T, G), X)
    assert failed.cpu().numpy()[0] == 1


@pytest.mark.parametrize("M,N,K,batch", [(300, 200, 100, 1), (129, 17, 34, 2), (520, 300, 778, 3), (64, 128, 16, 1)])
def test_dgemm_real_ragged_batched(T, M, N, K, batch):
    """traj_dgemm (the real DMMA GEMM of the planar 3M propagator) against NumPy: tails that are not
    multiples of the 128 x 128 tile or the 16-deep stage, alpha/beta, batches, B's leading dimension
    padded to 16 columns, C's to an even count."""
    import paper_2508_18468_b200 as P
    rng = np.random.default_rng(M + N + K)
    ldb = (N + 15) // 16 * 16
    ldc = N + (N & 1)
    lda = K + (K & 1)
    A = rng.standard_normal((batch, M, lda))
    B = rng.standard_normal((batch, K, ldb))
    C = rng.standard_normal((batch, M, ldc))
    want = 0.5 * np.einsum("bmk,bkn->bmn", A[:, :, :K], B[:, :, :N]) + 2.0 * C[:, :, :N]
    dA, dB, dC = dev(T, A), dev(T, B), dev(T, C)
    st = T.cuda.current_stream().cuda_stream
    r = P.lib().traj_dgemm(st, M, N, K, 0.5, dA.data_ptr(), lda, M * lda if batch > 1 else 0, dB.data_ptr(), ldb,
                           K * ldb if batch > 1 else 0, 2.0, dC.data_ptr(), ldc, M * ldc, batch)
    assert r == 0
    got = dC.cpu().numpy()[:, :, :N]
    assert np.abs(got - want).max() < 1e-12 * max(1.0, np.abs(want).max()) * K ** 0.5
    assert np.array_equal(dC.cpu().numpy()[:, :, N:], C[:, :, N:])      # padding untouched


def test_dgemm_rejects_bad_layouts(T):
    import paper_2508_18468_b200 as P
    st = T.cuda.current_stream().cuda_stream
    A = T.zeros(8, 8, dtype=T.float64, device="cuda")
    assert P.lib().traj_dgemm(st, 8, 8, 8, 1.0, A.data_ptr(), 7, 0, A.data_ptr(), 8, 0, 0.0, A.data_ptr(), 8, 0, 1) == 1
    assert P.lib().traj_dgemm(st, 8, 8, 8, 1.0, A.data_ptr(), 8, 0, A.data_ptr(), 8, 0, 0.0, A.data_ptr(), 8, 0, 1) == 1
