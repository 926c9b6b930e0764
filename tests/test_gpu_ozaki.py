"""The exact modular complex products on the INT8 tensor cores (csrc/igemm.cu, csrc/ozaki.cu) through
the C-ABI: traj_igemm against NumPy int64 (exact, both epilogues, ragged tiles, the upper-tile and
triangular-B skips), traj_zgemm_ozaki against an extended-precision (long double) product with the
error bound the scheme guarantees (every input represented to 2^-beta of its row / column 2-norm,
products exact): plain, conjugated (the Gram form U^dag U), upper-only, triangular B, rows spanning
many decades, zero rows and a banded propagator-like operand whose entries decay to 1e-300."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BETA = {4: 14, 6: 22, 8: 29, 10: 37, 12: 44, 14: 51, 16: 57, 18: 61}


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


@pytest.mark.parametrize("M,N,K,batch,mod,flags", [(300, 520, 1000, 2, False, 0), (128, 256, 128, 1, False, 0),
                                                   (300, 520, 1000, 3, True, 0), (700, 700, 700, 1, False, 1),
                                                   (400, 700, 700, 1, False, 2), (1, 33, 16, 1, True, 0),
                                                   (600, 600, 2100, 2, True, 1), (520, 600, 600, 3, True, 2)])
def test_igemm_exact(T, M, N, K, batch, mod, flags):
    import paper_2508_18468_b200 as P
    rng = np.random.default_rng(M * 7 + N + K)
    lda = (K + 15) // 16 * 16
    ldc = (N + 15) // 16 * 16
    A = rng.integers(-128, 128, size=(batch, M, lda), dtype=np.int8)
    B = rng.integers(-128, 128, size=(batch, N, lda), dtype=np.int8)
    if flags & 2:
        for n in range(N):
            B[:, n, n + 1:] = 0
    want = np.einsum("zmk,znk->zmn", A[:, :, :K].astype(np.int64), B[:, :, :K].astype(np.int64))
    mods = np.array([251, 256, 193], dtype=np.int32)
    dA, dB = dev(T, A), dev(T, B)
    dC = T.zeros((batch, M, ldc), dtype=T.uint8 if mod else T.int32, device="cuda")
    dm = dev(T, mods)
    st = T.cuda.current_stream().cuda_stream
    r = P.lib().traj_igemm(st, M, N, K, dA.data_ptr(), lda, M * lda, dB.data_ptr(), lda, N * lda, dC.data_ptr(), ldc,
                           M * ldc, batch, dm.data_ptr() if mod else None, 3, flags)
    assert r == 0
    got = dC.cpu().numpy()[:, :, :N].astype(np.int64)
    if mod:
        want = np.stack([want[z] % mods[z % 3] for z in range(batch)])
    if flags & 1:   # only tiles meeting the upper triangle are written
        for m in range(M):
            for z in range(batch):
                lo = (m // 128) * 128
                keep = np.arange(N) // 256 * 256 + 255 >= lo
                got[z, m, ~keep] = want[z, m, ~keep]
    assert np.array_equal(got, want)


def test_igemm_rejects_bad_layouts(T):
    import paper_2508_18468_b200 as P
    st = T.cuda.current_stream().cuda_stream
    A = T.zeros(64, 64, dtype=T.int8, device="cuda")
    C = T.zeros(64, 64, dtype=T.int32, device="cuda")
    lib = P.lib()
    assert lib.traj_igemm(st, 64, 64, 64, A.data_ptr(), 40, 0, A.data_ptr(), 64, 0, C.data_ptr(), 64, 0, 1, None, 1, 0) == 1
    assert lib.traj_igemm(st, 64, 64, 0, A.data_ptr(), 64, 0, A.data_ptr(), 64, 0, C.data_ptr(), 64, 0, 1, None, 1, 0) == 1
    assert lib.traj_igemm(st, 64, 64, 64, A.data_ptr(), 64, 0, A.data_ptr(), 64, 0, C.data_ptr(), 8, 0, 1, None, 1, 0) == 1


def _ld(x):
    return x.astype(np.clongdouble)


def _bound(opA_mat, B, C_ref, s):
    """Error bound of the scheme: |dC_ij| <= 2^-beta (nu_a_i |b_j|_1 + nu_b_j |a_i|_1) (x4 margin for the
    complex parts) + the final rounding of C to FP64."""
    a = np.abs(opA_mat.real) + np.abs(opA_mat.imag)
    b = np.abs(B.real) + np.abs(B.imag)
    nua = np.sqrt((a ** 2).sum(1))
    nub = np.sqrt((b ** 2).sum(0))
    l1a = a.sum(1)
    l1b = b.sum(0)
    return 4.0 * 2.0 ** -BETA[s] * (nua[:, None] * l1b[None, :] + nub[None, :] * l1a[:, None]) + \
        4.0 * 2.0 ** -53 * np.abs(C_ref).astype(np.float64)


def _rand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _run(T, opA, A, B, s, flags=0, M=None):
    import paper_2508_18468_b200 as P
    K, N = B.shape
    if M is None:
        M = A.shape[1] if opA else A.shape[0]
    dA, dB = dev(T, A), dev(T, B)
    dC = T.full((M, N), complex(7.0, 7.0), dtype=T.complex128, device="cuda")
    st = T.cuda.current_stream().cuda_stream
    r = P.lib().traj_zgemm_ozaki(st, opA, M, N, K, dA.data_ptr(), A.shape[1], dB.data_ptr(), N, dC.data_ptr(), N, s,
                                 flags)
    assert r == 0, P.lib().traj_last_error(None)
    return dC.cpu().numpy()


@pytest.mark.parametrize("M,N,K", [(300, 200, 100), (129, 17, 534), (520, 300, 778), (16, 16, 16), (257, 513, 1300)])
@pytest.mark.parametrize("s", [8, 16, 18])
def test_zgemm_ozaki_matches_extended_precision(T, M, N, K, s):
    rng = np.random.default_rng(M + 3 * N + 5 * K + s)
    A = _rand(rng, M, K) * (10.0 ** rng.integers(-6, 7, size=(M, 1)))   # rows spanning 12 decades
    B = _rand(rng, K, N) * (10.0 ** rng.integers(-6, 7, size=(1, N)))
    A[M // 2] = 0.0
    ref = _ld(A) @ _ld(B)
    got = _run(T, 0, A, B, s)
    err = np.abs(got - ref.astype(np.complex128))
    assert (err <= _bound(A, B, ref, s)).all()
    assert np.all(got[M // 2] == 0)
    if s >= 16:   # at 16 moduli the result is as accurate as an FP64 GEMM's (here: within 2^-50 relative)
        assert (err <= 2.0 ** -50 * (np.abs(A) @ np.abs(B))).all()


@pytest.mark.parametrize("N,K", [(200, 300), (300, 1000), (64, 5000)])
def test_zgemm_ozaki_gram_form(T, N, K):
    """A^dag B and the Gram A^dag A (upper only) with orthonormal-ish columns, as in CholeskyQR."""
    rng = np.random.default_rng(N + K)
    A, _ = np.linalg.qr(_rand(rng, K, N))
    A = A + 1e-7 * _rand(rng, K, N)
    B = _rand(rng, K, N)
    ref = _ld(A).conj().T @ _ld(B)
    got = _run(T, 1, A, B, 16)
    assert (np.abs(got - ref.astype(np.complex128)) <= _bound(A.conj().T, B, ref, 16)).all()
    G = _run(T, 1, A, A, 16, flags=16)
    Gref = (_ld(A).conj().T @ _ld(A)).astype(np.complex128)
    iu = np.triu_indices(N)
    assert np.abs(G[iu] - Gref[iu]).max() < 1e-16 * K ** 0.5
    il = np.tril_indices(N, -1)
    assert np.all(G[il] == complex(7.0, 7.0))   # below the diagonal untouched
    # E = G - I to high relative accuracy (what the second CholeskyQR pass needs)
    E = G - np.eye(N)
    Eref = Gref - np.eye(N)
    assert np.abs(E[iu] - Eref[iu]).max() <= 1e-3 * np.abs(Eref[iu]).max() + 1e-17


def test_zgemm_ozaki_triangular_b(T):
    rng = np.random.default_rng(5)
    L, N = 700, 300
    U = _rand(rng, L, N)
    X = np.triu(_rand(rng, N, N))
    ref = _ld(U) @ _ld(X)
    got = _run(T, 0, U, X, 16, flags=4)
    assert (np.abs(got - ref.astype(np.complex128)) <= _bound(U, X, ref, 16)).all()


def test_zgemm_ozaki_banded_propagator_operand(T):
    """K = exp(-i H dt) rows on a ring: entries decay from ~1 to below 1e-300 -- the fixed-point rows
    drop what FP64 could not add anyway; the product matches at FP64 accuracy."""
    from scipy.linalg import expm
    L, N = 512, 256
    H = np.zeros((L, L))
    for i in range(L):
        H[i, (i + 1) % L] = H[(i + 1) % L, i] = -1.0
    Kp = expm(-1j * 0.05 * H)
    rng = np.random.default_rng(9)
    U, _ = np.linalg.qr(_rand(rng, L, N))
    ref = _ld(Kp) @ _ld(U)
    got = _run(T, 0, Kp, U, 16)
    assert np.abs(got - ref.astype(np.complex128)).max() < 4e-17


def test_zgemm_ozaki_rejects(T):
    import paper_2508_18468_b200 as P
    st = T.cuda.current_stream().cuda_stream
    A = T.zeros(16, 16, dtype=T.complex128, device="cuda")
    lib = P.lib()
    assert lib.traj_zgemm_ozaki(st, 0, 16, 16, 16, A.data_ptr(), 16, A.data_ptr(), 16, A.data_ptr(), 16, 7, 0) == 1
    assert lib.traj_zgemm_ozaki(st, 2, 16, 16, 16, A.data_ptr(), 16, A.data_ptr(), 16, A.data_ptr(), 16, 16, 0) == 1
    assert lib.traj_zgemm_ozaki(st, 0, 16, 16, 16, A.data_ptr(), 8, A.data_ptr(), 16, A.data_ptr(), 16, 16, 0) == 1


# ---- the modular products inside the trajectory step (env thresholds lowered so small lattices take
# ---- the path the full-size configs take), in lockstep with the oracle

@pytest.fixture
def oz_small(monkeypatch):
    monkeypatch.setenv("TRAJ_PLANAR_MIN_N", "64")      # the modular K U / Gram / TRMM from N = 64 on
    monkeypatch.setenv("TRAJ_OZAKI_PROJ_MIN", "1")     # the modular rank-k products at any click count
    monkeypatch.delenv("TRAJ_OZAKI", raising=False)


def _oz_on(P, *args, **kw):
    g = P.Trajectories(*args, **kw)
    assert g.ozaki_info()[:2] == (True, True)
    return g


def test_step_on_modular_path_projective_matches_oracle(T, oz_small):
    import paper_2508_18468_b200 as P
    from test_gpu_parity import lockstep
    _oz_on(P, 300, 1, "projective", [2.0, 0.6])
    lockstep(P, 300, 1, "projective", [2.0, 0.6], 30, 5, [np.arange(150), np.arange(37, 211)], seed=7)


def test_step_on_modular_path_homodyne_and_2d_match_oracle(T, oz_small):
    import paper_2508_18468_b200 as P
    import workloads
    from test_gpu_parity import lockstep
    lockstep(P, 200, 1, "homodyne", [0.1, 1.0, 3.0], 60, 20, [np.arange(100), np.arange(13)], seed=3, traj_base=5)
    A, B = workloads.strips_2d(16, 12)
    lockstep(P, 16, 12, "projective", [2.86, 5.72], 30, 10, [workloads.columns(16, 12, 0, 8)], seed=5, mi=(A, B))


def test_modular_cqr2_fallback_is_full_precision(T, oz_small):
    """An ill-conditioned state (kappa ~ 1e5) makes the second pass take the full factorisation: the
    gated 16-moduli TRMM then overwrites the cheap first-order correction."""
    import torch
    import paper_2508_18468_b200 as P
    from oracle import gaussian
    L, N = 200, 100
    U = workloads_random(L, N, 3)
    U[:, 1] = U[:, 0] + 1e-5 * U[:, 1]
    c = _oz_on(P, L, 1, "homodyne", [0.0])
    c.set_state(0, torch.from_numpy(U).cuda())
    c.orthonormalize()
    assert c.cqr2_fallbacks() == 1
    Ug = c.get_state(0).cpu().numpy()
    assert np.abs(Ug.conj().T @ Ug - np.eye(N)).max() < 1e-12
    assert np.abs(c.correlation(0).cpu().numpy() - gaussian.correlation(gaussian.orthonormalize(U))).max() < 1e-9


@pytest.mark.parametrize("low", ["8", "6", "0"])
def test_modular_correction_tiers(T, oz_small, monkeypatch, low):
    """The first-order second pass dst = src + src D on the modular path picks its modulus count on the
    device from the column norms of D = X - I (low tier when all are <= 2^(beta_low - 55.5) / N, else the
    standard count, else the full product): every tier must reproduce the full-precision src X to
    rounding and leave U orthonormal.  Inputs with two nearly parallel columns span the well-conditioned case (low tier) to
    deviations above the low threshold (the threshold itself is replayed here from the Gram)."""
    import ctypes
    import torch
    import paper_2508_18468_b200 as P
    L, N = 256, 128
    rng = np.random.default_rng(11)
    Q, _ = np.linalg.qr(rng.standard_normal((L, N)) + 1j * rng.standard_normal((L, N)))
    mods = (ctypes.c_int32 * 32)()
    beta = ctypes.c_int32(0)
    ch, cl, M = (ctypes.c_double * 32)(), (ctypes.c_double * 32)(), ctypes.c_double()
    devs = []
    for delta in (1.0, 2e-2, 5e-3, 2.5e-3):
        U0 = Q.copy()
        U0[:, 1] = Q[:, 0] + delta * Q[:, 1]       # kappa ~ 2 / delta: the first pass leaves ~ kappa^2 eps
        U0 = np.ascontiguousarray(U0)
        out = {}
        fell_back = False
        for mode in ("tiered", "full"):
            monkeypatch.setenv("TRAJ_OZAKI_CORR_LOW", low)
            monkeypatch.setenv("TRAJ_OZAKI_CORR_MODULI", "10" if mode == "tiered" else "0")
            c = _oz_on(P, L, 1, "homodyne", [0.0])
            c.set_state(0, torch.from_numpy(U0).cuda())
            c.orthonormalize()
            fell_back |= c.cqr2_fallbacks() != 0
            dev = float(c.gram_deviation()[0])
            out[mode] = c.get_state(0).cpu().numpy()
        if fell_back:        # the full factorisation's own path (test_modular_cqr2_fallback_is_full_precision)
            continue
        devs.append(dev)
        print("delta", delta, "max|G2 - I|", dev)
        Ug = out["tiered"]
        assert np.abs(Ug.conj().T @ Ug - np.eye(N)).max() < 5e-15
        assert np.abs(Ug - out["full"]).max() < 2e-15
    # the sweep must straddle the low tier's threshold: |D col| <= sqrt(N) max|E| from below, >= max|E| / 2
    # from above
    if int(low) > 0:
        assert P.lib().traj_ozaki_constants(int(low), mods, ctypes.byref(beta), ch, cl, ctypes.byref(M)) == 0
        dmax = 2.0 ** (beta.value - 55.5) / N
        assert min(devs) * np.sqrt(N) < dmax
        if low == "6":
            assert max(devs) / 2 > dmax


def workloads_random(L, N, seed):
    from workloads import random_matrix
    return random_matrix(L, N, seed)


def test_modular_step_matches_dmma_step(T, monkeypatch):
    """The same c3-shaped trajectory (L = 2048, projective) on the modular path and on the DMMA kernels:
    identical clicks, C within 1e-12 after 4 steps."""
    import paper_2508_18468_b200 as P
    monkeypatch.setenv("TRAJ_OZAKI_PROJ_MIN", "1")
    a = P.Trajectories(2048, 1, "projective", [0.3, 1.5], seed=1)
    monkeypatch.setenv("TRAJ_OZAKI", "0")
    b = P.Trajectories(2048, 1, "projective", [0.3, 1.5], seed=1)
    assert a.ozaki_info()[0] and not b.ozaki_info()[0]
    for _ in range(4):
        a.step(1)
        b.step(1)
        for t in range(2):
            assert a.last_clicks(t) == b.last_clicks(t)
    for t in range(2):
        assert np.abs(a.correlation(t).cpu().numpy() - b.correlation(t).cpu().numpy()).max() < 1e-12


def test_modular_cholesky_levels_match_oracle(T, monkeypatch):
    """chol_inverse's large recursion levels on the modular path (threshold lowered to 128): the dense
    CholeskyQR passes of a homodyne trajectory in lockstep with the oracle, and the ill-conditioned
    second-pass fallback (conditional graph) at full precision."""
    import torch
    import paper_2508_18468_b200 as P
    from oracle import gaussian
    from test_gpu_parity import lockstep
    monkeypatch.setenv("TRAJ_PLANAR_MIN_N", "64")
    monkeypatch.setenv("TRAJ_CHOL_OZAKI_MIN", "128")
    lockstep(P, 600, 1, "homodyne", [0.3, 2.0], 20, 5, [np.arange(300), np.arange(41, 377)], seed=13)
    L, N = 600, 300
    U = workloads_random(L, N, 4)
    U[:, 7] = U[:, 3] + 1e-5 * U[:, 7]
    c = _oz_on(P, L, 1, "homodyne", [0.0])
    c.set_state(0, torch.from_numpy(U).cuda())
    c.orthonormalize()
    assert c.cqr2_fallbacks() == 1
    Ug = c.get_state(0).cpu().numpy()
    assert np.abs(Ug.conj().T @ Ug - np.eye(N)).max() < 1e-12
    assert np.abs(c.correlation(0).cpu().numpy() - gaussian.correlation(gaussian.orthonormalize(U))).max() < 1e-9


@pytest.mark.parametrize("protocol", ["homodyne", "projective"])
def test_modular_path_nan_trajectory_fails_alone(T, oz_small, protocol):
    """A trajectory whose state holds a NaN stays failed on the modular path (non-finite rows and
    columns come out as NaN, as an FP64 product's would) and does not disturb the other trajectory of
    the batch, which still matches the oracle."""
    import torch
    import paper_2508_18468_b200 as P
    from oracle import lattice
    from oracle.trajectory import OracleTrajectory
    L, gams, steps = 300, [1.0, 1.5], 6
    gpu = _oz_on(P, L, 1, protocol, gams, seed=3)
    U = gpu.get_state(0).cpu().numpy()
    U[17, 5] = np.nan
    gpu.set_state(0, torch.from_numpy(U).cuda())
    K = lattice.propagator_lattice(L, 1, 1.0, 0.05)
    o1 = OracleTrajectory(L, 1, protocol, gams[1], 0.05, seed=3, traj=1, K=K)
    gpu.step(steps)
    o1.step(steps)
    assert gpu.failed(0) and not gpu.failed(1)
    assert np.abs(gpu.correlation(1).cpu().numpy() - o1.correlation()).max() < 1e-10


# ---- the row-sharded step on the modular engine: K_g U as P chunk products whose
# ---- residues accumulate over the chunks at U's global column exponents, local modular Grams / TRMMs

@pytest.mark.parametrize("L,P_shards,protocol,gam,variant", [
    (480, 2, "projective", 2.0, "one_product"), (480, 3, "homodyne", 1.0, "chunks"),
    (512, 4, "projective", 0.7, "chunks"), (512, 8, "homodyne", 2.0, "one_product"),
    (512, 8, "projective", 3.0, "one_product"), (512, 2, "projective", 3.0, "serial_structured")])
def test_row_sharded_modular_step_matches_oracle_and_dmma(T, oz_small, monkeypatch, L, P_shards, protocol, gam,
                                                          variant):
    """Single-GPU emulation of P shards (Lp = 240, 160, 128, 64 rows: ragged against the 128-row tiles)
    on the modular path -- K_g U as one depth-L product of the gathered U's residues, or (chunks) as
    the P ring-ordered chunk products accumulated in the residue epilogue; the projective C_SS, rank-k
    update and structured pass-1 solve modular too (threshold lowered), the structured factor
    pipelined or (serial_structured) not -- against the same trajectory on the sharded DMMA kernels
    (TRAJ_OZAKI=0) and the oracle: identical clicks, C within 1e-12 of the DMMA step and 1e-10 of the
    oracle, S_A within 1e-8."""
    import paper_2508_18468_b200 as P
    from oracle import lattice
    from oracle.trajectory import OracleTrajectory
    if variant == "chunks":
        monkeypatch.setenv("TRAJ_SHARD_OZ_CHUNKS", "1")
    if variant == "serial_structured":
        monkeypatch.setenv("TRAJ_STRUCT_PIPELINE", "0")
    a = P.Trajectories(L, 1, protocol, [gam], seed=23, traj_base=1, shard_size=P_shards)
    assert a.ozaki_info() == (True, True, 16)
    monkeypatch.setenv("TRAJ_OZAKI", "0")
    b = P.Trajectories(L, 1, protocol, [gam], seed=23, traj_base=1, shard_size=P_shards)
    assert not b.ozaki_info()[0]
    o = OracleTrajectory(L, 1, protocol, gam, 0.05, seed=23, traj=1, K=lattice.propagator_lattice(L, 1, 1.0, 0.05))
    regions = [np.arange(L // 2), np.arange(37, 211)]
    for s in range(12):
        a.step(1)
        b.step(1)
        o.step(1)
        if protocol == "projective":
            assert a.last_clicks(0) == b.last_clicks(0) == (o.last_clicks[0].size, int(o.last_clicks[1].sum()))
        if s % 4 == 3:
            ca = a.correlation(0).cpu().numpy()
            assert np.abs(ca - b.correlation(0).cpu().numpy()).max() < 1e-12
            assert np.abs(ca - o.correlation()).max() < 1e-10
            for A in regions:
                assert abs(a.entropy(A)[0] - o.entropy(A)) < 1e-8
    U = a.get_state(0).cpu().numpy()
    assert np.abs(U.conj().T @ U - np.eye(L // 2)).max() < 1e-12
    assert not a.failed(0)
    a.close()
    b.close()


def test_row_sharded_modular_nccl_single_rank(T, oz_small):
    """The NCCL code path of the sharded modular step (a one-rank communicator: the global column
    exponents' allreduce, the chunk residues, the local Gram) against the unsharded modular handle."""
    import paper_2508_18468_b200 as P
    L = 232
    uid = P.traj_nccl_unique_id()
    a = P.Trajectories(L, 1, "projective", [3.0], seed=5, shard_size=1, shard_rank=0, nccl_id=uid)
    b = P.Trajectories(L, 1, "projective", [3.0], seed=5)
    assert a.ozaki_info() == b.ozaki_info() == (True, True, 16)
    a.step(10)
    b.step(10)
    assert a.last_clicks(0) == b.last_clicks(0)
    assert np.abs(a.correlation(0).cpu().numpy() - b.correlation(0).cpu().numpy()).max() < 1e-12
    U = a.get_state(0).cpu().numpy()
    assert np.abs(U.conj().T @ U - np.eye(L // 2)).max() < 1e-12
    a.close()
    b.close()
