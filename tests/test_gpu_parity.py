"""GPU path (through the C-ABI) vs the oracle on the same seeded Philox streams.

Bar (north star): C = U U^dag within 1e-10 absolute and S_A within 1e-8 over short runs;
projective click lists and outcomes identical.  Sizes span several 128 x 64 GEMM tiles
with ragged tails; configs c1 (full) and reduced c2/c4-shaped cases; full-size c3 checks
via closed forms and invariants that hold at any size."""
import numpy as np
import pytest

import workloads
from oracle import gaussian, lattice
from oracle.trajectory import OracleTrajectory

pytestmark = pytest.mark.gpu

C_TOL = 1e-10
S_TOL = 1e-8


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2508_18468_b200 import build
    build.build()
    import paper_2508_18468_b200 as P
    P.load_library()
    return P


def lockstep(P, Lx, Ly, protocol, gammas, steps, sample_every, regions, seed=0, traj_base=0, dt=0.05,
             mi=None, check_clicks=True):
    gpu = P.Trajectories(Lx, Ly, protocol, gammas, dt=dt, seed=seed, traj_base=traj_base)
    K = lattice.propagator_lattice(Lx, Ly, 1.0, dt)
    orc = [OracleTrajectory(Lx, Ly, protocol, g, dt, seed=seed, traj=traj_base + t, K=K)
           for t, g in enumerate(gammas)]
    worst_c = worst_s = 0.0
    clicks = 0
    for s in range(steps + 1):
        if s % sample_every == 0:
            for t, o in enumerate(orc):
                C = gpu.correlation(t).cpu().numpy()
                worst_c = max(worst_c, np.abs(C - o.correlation()).max())
            for A in regions:
                S = gpu.entropy(A)
                for t, o in enumerate(orc):
                    worst_s = max(worst_s, abs(S[t] - o.entropy(A)))
            if mi is not None:
                I = gpu.mutual_info(*mi)
                for t, o in enumerate(orc):
                    worst_s = max(worst_s, abs(I[t] - o.mutual_info(*mi)))
        if s == steps:
            break
        gpu.step(1)
        for t, o in enumerate(orc):
            o.step(1)
            if protocol == "projective" and check_clicks:
                nS, n1 = gpu.last_clicks(t)
                S_, occ = o.last_clicks
                assert (nS, n1) == (S_.size, int(occ.sum())), (s, t)
                clicks += nS
    for t in range(len(gammas)):
        assert not gpu.failed(t)
    assert worst_c < C_TOL, worst_c
    assert worst_s < S_TOL, worst_s
    return gpu, orc, clicks


def test_c1_projective_full(P):
    """configs[0]: L = 64, projective gamma = 0.5, 16 trajectories, 200 steps, S(half) every 10."""
    w = workloads.c1()
    _, _, clicks = lockstep(P, w.Lx, w.Ly, w.protocol, [w.gamma_of(t) for t in range(w.n_traj)], w.steps,
                            w.sample_every, [w.regions["half"]], seed=w.seed)
    assert clicks > 100


def test_projective_ragged_many_clicks(P):
    """L = 300 (N = 150: 3 ragged 64-wide tiles), p = gamma dt = 0.1: ~30 clicks per step."""
    lockstep(P, 300, 1, "projective", [2.0, 0.6], 30, 5, [np.arange(150), np.arange(37, 211)], seed=7)


def test_homodyne_1d_ragged(P):
    """c2-shaped (homodyne, gamma sweep) at L = 200."""
    lockstep(P, 200, 1, "homodyne", [0.1, 1.0, 3.0], 100, 20, [np.arange(100), np.arange(13)], seed=3,
             traj_base=5)


def test_homodyne_2d_mutual_information(P):
    """c4-shaped (2d torus, checkerboard, homodyne, MI between strips) at 12 x 8."""
    A, B = workloads.strips_2d(12, 8)
    lockstep(P, 12, 8, "homodyne", [0.5, 3.0], 60, 20, [workloads.columns(12, 8, 0, 6)], seed=11, mi=(A, B))


def test_projective_2d(P):
    """c5-shaped (2d, projective near the per-site critical rate) at 10 x 10."""
    A, B = workloads.strips_2d(10, 10)
    lockstep(P, 10, 10, "projective", [2.86, 5.72], 40, 10, [workloads.columns(10, 10, 0, 5)], seed=5, mi=(A, B))


def test_every_site_measured(P):
    """gamma dt = 1: N occupied outcomes, C diagonal 0/1, S = 0 after the step."""
    L = 96
    g = P.Trajectories(L, 1, "projective", [20.0, 20.0], dt=0.05, seed=2)
    g.step(3)
    for t in range(2):
        nS, n1 = g.last_clicks(t)
        assert nS == L and n1 == L // 2
        C = g.correlation(t).cpu().numpy()
        assert np.abs(C - np.diag(np.diag(C))).max() < 1e-12
        d = np.diag(C).real
        assert np.all((np.abs(d) < 1e-12) | (np.abs(d - 1) < 1e-12))
    assert np.all(np.abs(g.entropy(np.arange(L // 2))) < 1e-9)


def test_set_state_orthonormalize_matches_householder(P):
    """CholeskyQR2 of an arbitrary full-rank U spans the same subspace as Householder QR."""
    import torch
    L, N = 200, 100
    g = P.Trajectories(L, 1, "homodyne", [0.0], seed=0)
    U = workloads.random_matrix(L, N, 21)
    g.set_state(0, torch.from_numpy(U).cuda())
    g.orthonormalize()
    Ug = g.get_state(0).cpu().numpy()
    assert np.abs(Ug.conj().T @ Ug - np.eye(N)).max() < 1e-13
    Q = gaussian.orthonormalize(U)
    assert np.abs(g.correlation(0).cpu().numpy() - gaussian.correlation(Q)).max() < 1e-12


def test_free_evolution_closed_form_full_c3(P):
    """configs[2] size (L = 16384, N = 8192), gamma = 0: n_i(t) = 1/2 + (-1)^i/(2L) sum_m cos(4t cos(2 pi m/L))
    after 10 steps; Tr C = N; the step keeps U^dag U = 1."""
    L, steps, dt = 16384, 10, 0.05
    g = P.Trajectories(L, 1, "projective", [0.0], dt=dt, seed=0)
    g.step(steps)
    n = g.occupations()[0].cpu().numpy()
    m = np.arange(L)
    want = 0.5 + 0.5 * (-1.0) ** m * np.mean(np.cos(4 * steps * dt * np.cos(2 * np.pi * m / L)))
    assert np.abs(n - want).max() < 1e-12
    assert abs(n.sum() - L // 2) < 1e-8


def test_projective_full_c3_invariants(P):
    """configs[2] (L = 16384, gamma = 0.3): after a step every clicked site has n in {0, 1},
    the particle number is N, U stays orthonormal, and S_A = S_complement."""
    import torch
    from paper_2508_18468_b200 import traj_zgemm
    w = workloads.c3()
    g = P.Trajectories(w.Lx, 1, "projective", list(w.gammas), dt=w.dt, seed=w.seed)
    g.step(2)
    nS, n1 = g.last_clicks(0)
    assert 150 < nS < 350
    from oracle.philox import site_uniforms
    u0, _ = site_uniforms(w.L, 1, 0, w.seed)
    S = np.nonzero(u0 < w.gammas[0] * w.dt)[0]
    assert S.size == nS
    n = g.occupations()[0].cpu().numpy()
    ns = n[S]
    assert np.all((np.abs(ns) < 1e-10) | (np.abs(ns - 1) < 1e-10))
    assert int(np.round(ns.sum())) == n1
    assert abs(n.sum() - w.N) < 1e-7
    U = g.get_state(0)
    G = torch.zeros((w.N, w.N), dtype=torch.complex128, device="cuda")
    traj_zgemm(1, 0, U, U, G)
    G -= torch.eye(w.N, dtype=torch.complex128, device="cuda")
    assert G.abs().max().item() < 1e-12
    del G, U
    A = np.arange(w.L // 8)
    Ac = np.arange(w.L // 8, w.L)
    sa, sc = g.entropy(A)[0], g.entropy(Ac)[0]
    assert abs(sa - sc) < 1e-8


def test_free_evolution_closed_form_full_c5(P):
    """configs[4] size (2d 160 x 160, N = 12800), gamma = 0, checkerboard start: after 5 steps
    n = 1/2 + (-1)^(x+y)/2 s(t)^2 with s(t) = (1/160) sum_m cos(4t cos(2 pi m/160)) -- the 2d
    Kronecker K as planar products and CholeskyQR at full size.  Tr C = N."""
    Lx = Ly = 160
    steps, dt = 5, 0.05
    g = P.Trajectories(Lx, Ly, "projective", [0.0], dt=dt, seed=0)
    g.step(steps)
    n = g.occupations()[0].cpu().numpy()
    m = np.arange(Lx)
    s_t = np.mean(np.cos(4 * steps * dt * np.cos(2 * np.pi * m / Lx)))
    ys, xs = np.divmod(np.arange(Lx * Ly), Lx)
    want = 0.5 + 0.5 * (-1.0) ** (xs + ys) * s_t ** 2
    assert np.abs(n - want).max() < 1e-12
    assert abs(n.sum() - Lx * Ly // 2) < 1e-7
    g.close()


def test_projective_full_c5_invariants(P):
    """configs[4] (160 x 160, projective gamma = 2.86, ~3660 clicks per step): after two steps every
    clicked site has n in {0, 1} and the occupied count matches, the particle number is N, U stays
    orthonormal, and S_A = S_complement for the strip A = x in [0, 40)."""
    import torch
    from paper_2508_18468_b200 import traj_zgemm
    w = workloads.c5()
    g = P.Trajectories(w.Lx, w.Ly, "projective", list(w.gammas), dt=w.dt, seed=w.seed)
    g.step(2)
    nS, n1 = g.last_clicks(0)
    assert 3200 < nS < 4200
    from oracle.philox import site_uniforms
    u0, _ = site_uniforms(w.L, 1, 0, w.seed)
    S = np.nonzero(u0 < w.gammas[0] * w.dt)[0]
    assert S.size == nS
    n = g.occupations()[0].cpu().numpy()
    ns = n[S]
    assert np.all((np.abs(ns) < 1e-10) | (np.abs(ns - 1) < 1e-10))
    assert int(np.round(ns.sum())) == n1
    assert abs(n.sum() - w.N) < 1e-7
    U = g.get_state(0)
    G = torch.zeros((w.N, w.N), dtype=torch.complex128, device="cuda")
    traj_zgemm(1, 0, U, U, G)
    G -= torch.eye(w.N, dtype=torch.complex128, device="cuda")
    assert G.abs().max().item() < 1e-12
    del G, U
    A = workloads.columns(w.Lx, w.Ly, 0, w.Lx // 4)
    Ac = np.setdiff1d(np.arange(w.L), A)
    assert abs(g.entropy(A)[0] - g.entropy(Ac)[0]) < 1e-8
    g.close()


def test_c2_full_size_homodyne_lockstep(P):
    """configs[1] at full size (1d L = 2048, N = 1024, homodyne, gamma in {0.1, 0.3, 1.0} as one
    batch of three trajectories): the planar defaults with trajectory batching, 50 steps in lockstep
    with the oracle (>= 50-step windows); C and S(half) every 10 steps."""
    w = workloads.c2()
    gams = list(w.gammas)
    lockstep(P, w.Lx, w.Ly, w.protocol, gams, 50, 10, [w.regions["half"]], seed=w.seed)


def test_c4_full_size_homodyne_mutual_information(P):
    """configs[3] at full size (2d 64 x 64, N = 2048, homodyne, all 8 gammas of the sweep as one batch
    of trajectories): 4 steps in lockstep with the oracle including I2 between the 16 x 64 strips."""
    w = workloads.c4()
    gams = list(w.gammas)
    A, B = w.regions["mi"]
    lockstep(P, w.Lx, w.Ly, w.protocol, gams, 4, 4, [A], seed=w.seed, mi=(A, B))


@pytest.mark.parametrize("levels", [1, 2, 3])
@pytest.mark.parametrize("Lx,Ly,protocol,gams", [(208, 1, "projective", [2.0]), (208, 1, "homodyne", [1.0, 0.3]),
                                               (12, 12, "projective", [3.0, 1.0]), (12, 12, "homodyne", [1.5])])
def test_strassen_propagator_matches_oracle(P, monkeypatch, Lx, Ly, protocol, gams, levels):
    """Strassen on each planar real product of K U (csrc/planar.cu strassen_*), one level (seven
    half-size products), two (49 quarter-size ones) and three (343 eighth-size ones, one trajectory;
    with two trajectories it falls back to two): the same state as the plain planar products (1e-12)
    and the oracle (1e-10) -- 1d and 2d (Kronecker K), one launch for all products and trajectories."""
    L, steps = Lx * Ly, 10
    monkeypatch.setenv("TRAJ_PLANAR_MIN_N", "0")
    monkeypatch.setenv("TRAJ_STRASSEN_MIN_N", "0")
    monkeypatch.setenv("TRAJ_OZAKI", "0")   # the DMMA planar products (the modular ones: test_gpu_ozaki.py)
    monkeypatch.setenv("TRAJ_STRASSEN_LEVELS", str(levels))
    a = P.Trajectories(Lx, Ly, protocol, gams, seed=17)
    monkeypatch.setenv("TRAJ_STRASSEN", "0")
    b = P.Trajectories(Lx, Ly, protocol, gams, seed=17)
    K = lattice.propagator_lattice(Lx, Ly, 1.0, 0.05)
    orc = [OracleTrajectory(Lx, Ly, protocol, g, 0.05, seed=17, traj=t, K=K) for t, g in enumerate(gams)]
    for s in range(steps):
        a.step(1)
        b.step(1)
        for o in orc:
            o.step(1)
    for t, o in enumerate(orc):
        Ca, Cb = a.correlation(t).cpu().numpy(), b.correlation(t).cpu().numpy()
        assert np.abs(Ca - Cb).max() < 1e-12
        assert np.abs(Ca - o.correlation()).max() < C_TOL
        if protocol == "projective":
            assert a.last_clicks(t) == b.last_clicks(t)


@pytest.mark.parametrize("levels,shards,protocol", [(1, 2, "projective"), (2, 2, "homodyne"), (1, 4, "homodyne"),
                                                   (2, 4, "projective")])
def test_row_sharded_strassen_chunks_match_oracle(P, monkeypatch, levels, shards, protocol):
    """Strassen on every K-chunk product K_g[:, s] U_s of the row-sharded propagate (the chunk operands
    formed once per shard, the recombination accumulating over the ring-ordered chunks): the same state
    as the plain chunk products (1e-12) and the oracle (1e-10), P = 2 and 4 emulated shards."""
    L, steps, gam = 256, 8, (3.0 if protocol == "projective" else 1.0)
    monkeypatch.setenv("TRAJ_PLANAR_MIN_N", "0")
    monkeypatch.setenv("TRAJ_STRASSEN_MIN_N", "0")
    monkeypatch.setenv("TRAJ_OZAKI", "0")   # the DMMA planar products (the modular ones: test_gpu_ozaki.py)
    monkeypatch.setenv("TRAJ_STRASSEN_LEVELS", str(levels))
    a = P.Trajectories(L, 1, protocol, [gam], seed=19, shard_size=shards)
    monkeypatch.setenv("TRAJ_STRASSEN", "0")
    b = P.Trajectories(L, 1, protocol, [gam], seed=19, shard_size=shards)
    o = OracleTrajectory(L, 1, protocol, gam, 0.05, seed=19, traj=0, K=lattice.propagator_lattice(L, 1, 1.0, 0.05))
    for s in range(steps):
        a.step(1)
        b.step(1)
        o.step(1)
    Ca, Cb = a.correlation(0).cpu().numpy(), b.correlation(0).cpu().numpy()
    assert np.abs(Ca - Cb).max() < 1e-12
    assert np.abs(Ca - o.correlation()).max() < C_TOL
    if protocol == "projective":
        assert a.last_clicks(0) == b.last_clicks(0) == (o.last_clicks[0].size, int(o.last_clicks[1].sum()))


@pytest.mark.parametrize("block,shards,batched", [(128, 1, "1"), (64, 1, "1"), (64, 2, "1"), (48, 1, "1"),
                                                  (64, 1, "0"), (64, 2, "0")])
def test_structured_pass1_matches_dense_factorisation(P, monkeypatch, block, shards, batched):
    """CholeskyQR pass 1 of a projective step on the structure of G = I - V^dag V (csrc/structchol.cu):
    the same orthonormalised state as the dense Gram / Cholesky / TRMM pass (1e-12) and the oracle
    (1e-10), batched trajectories with different click counts, column blocks with a ragged tail
    (N = 350), and through the row-sharded emulation; both the batched factor (every block from its
    own S_c = I - sum_{d<c} V_d V_d^dag) and the sequential Woodbury chain (TRAJ_STRUCT_BATCHED=0)."""
    L, steps = 700, 12
    gams = [1.5, 0.8] if shards == 1 else [1.5]
    monkeypatch.setenv("TRAJ_STRUCT_B", str(block))
    monkeypatch.setenv("TRAJ_STRUCT_BATCHED", batched)
    a = P.Trajectories(L, 1, "projective", gams, seed=21, shard_size=shards)
    monkeypatch.setenv("TRAJ_STRUCT_CHOL", "0")
    b = P.Trajectories(L, 1, "projective", gams, seed=21, shard_size=shards)
    K = lattice.propagator_lattice(L, 1, 1.0, 0.05)
    orc = [OracleTrajectory(L, 1, "projective", g, 0.05, seed=21, traj=t, K=K) for t, g in enumerate(gams)]
    for s in range(steps):
        a.step(1)
        b.step(1)
        for t, o in enumerate(orc):
            o.step(1)
            assert a.last_clicks(t) == b.last_clicks(t) == (o.last_clicks[0].size, int(o.last_clicks[1].sum()))
    for t, o in enumerate(orc):
        Ca, Cb = a.correlation(t).cpu().numpy(), b.correlation(t).cpu().numpy()
        assert np.abs(Ca - Cb).max() < 1e-12
        assert np.abs(Ca - o.correlation()).max() < C_TOL
        U = a.get_state(t).cpu().numpy()
        assert np.abs(U.conj().T @ U - np.eye(L // 2)).max() < 1e-12
        assert not a.failed(t)


def test_cqr2_first_order_second_pass_matches_full(P):
    """The second CQR pass uses R2^-1 = I - triu(E,1) - diag(E)/2 (exact to O(N|E|^2));
    the result equals the full Cholesky second pass, and an ill-conditioned state falls back."""
    import os
    import torch
    args = (200, 1, "homodyne", [1.0, 3.0])
    a = P.Trajectories(*args, seed=4)
    os.environ["TRAJ_CQR2_FULL"] = "1"
    try:
        b = P.Trajectories(*args, seed=4)
    finally:
        del os.environ["TRAJ_CQR2_FULL"]
    a.step(40)
    b.step(40)
    assert a.cqr2_fallbacks() == 0
    for t in range(2):
        assert np.abs(a.correlation(t).cpu().numpy() - b.correlation(t).cpu().numpy()).max() < 1e-12
    # kappa ~ 1e5: pass 1 leaves |E| ~ 1e-6, so the second pass must factor G2 fully
    L, N = 200, 100
    U = workloads.random_matrix(L, N, 3)
    U[:, 1] = U[:, 0] + 1e-5 * U[:, 1]
    c = P.Trajectories(L, 1, "homodyne", [0.0])
    c.set_state(0, torch.from_numpy(U).cuda())
    c.orthonormalize()
    assert c.cqr2_fallbacks() == 1
    Ug = c.get_state(0).cpu().numpy()
    assert np.abs(Ug.conj().T @ Ug - np.eye(N)).max() < 1e-12
    assert np.abs(c.correlation(0).cpu().numpy() - gaussian.correlation(gaussian.orthonormalize(U))).max() < 1e-9


def test_projective_blocked_sampler_many_panels(P):
    """gamma dt = 0.5 at L = 400: ~200 clicks per step, i.e. 4 panels of the blocked sampler
    (in-panel sequential decisions + GEMM trailing updates) against the oracle's Eq. (A1)/(A2)."""
    _, _, clicks = lockstep(P, 400, 1, "projective", [10.0, 6.0], 12, 3, [np.arange(200)], seed=9)
    assert clicks > 12 * 250


def test_trajectory_parallel_ensemble_matches_oracle_average(P):
    """a5: ensemble statistics of a gamma sweep (ids folded with gamma), run in batches with
    traj_base offsets, equal the oracle's per-trajectory values averaged the same way."""
    from paper_2508_18468_b200.ensemble import run_ensemble
    w = workloads.Workload("mini", 32, 1, "projective", (0.5, 3.0), n_traj_per_gamma=3, steps=30,
                           sample_every=10, regions={"half": np.arange(16)})
    res = run_ensemble(w, 30, 10, {"half": ("entropy", np.arange(16))}, max_batch=4)
    K = lattice.propagator_lattice(32, 1, 1.0, 0.05)
    vals = np.zeros((w.n_traj, 4))
    for tau in range(w.n_traj):
        o = OracleTrajectory(32, 1, "projective", w.gamma_of(tau), 0.05, seed=0, traj=tau, K=K)
        for k in range(4):
            vals[tau, k] = o.entropy(np.arange(16))
            if k < 3:
                o.step(10)
    for g in range(2):
        x = vals[g * 3:(g + 1) * 3]
        assert np.all(res.count["half"][g] == 3)
        assert np.abs(res.mean["half"][g] - x.mean(axis=0)).max() < 1e-8


@pytest.mark.parametrize("P_shards,protocol,gamma", [(2, "projective", 4.0), (4, "homodyne", 1.0),
                                                     (4, "projective", 1.0)])
def test_row_sharded_step_matches_oracle(P, P_shards, protocol, gamma):
    """Row-sharded K and U, single-GPU emulation of P shards: allgather of U,
    local K_g U, global-site Philox, gathered clicks with replicated sampling, all-reduced Gram.
    Same trajectory as the oracle; entropies through both the gathered-rows (|A| <= N) and the
    all-reduced-Gram (|A| > N) paths."""
    L = 256
    g = P.Trajectories(L, 1, protocol, [gamma], seed=13, traj_base=2, shard_size=P_shards)
    assert (g.shard_size, g.local_shards, g.rows) == (P_shards, P_shards, L)
    K = lattice.propagator_lattice(L, 1, 1.0, 0.05)
    o = OracleTrajectory(L, 1, protocol, gamma, 0.05, seed=13, traj=2, K=K)
    regions = [np.arange(L // 2), np.arange(37, 77), np.arange(0, L, 3)[:150], np.arange(200)]
    for s in range(16):
        g.step(1)
        o.step(1)
        if protocol == "projective":
            assert g.last_clicks(0) == (o.last_clicks[0].size, int(o.last_clicks[1].sum()))
        if s % 5 == 4:
            assert np.abs(g.correlation(0).cpu().numpy() - o.correlation()).max() < C_TOL
            for A in regions:
                assert abs(g.entropy(A)[0] - o.entropy(A)) < S_TOL
    n = g.occupations()[0].cpu().numpy()
    assert np.abs(n - gaussian.occupations(o.U)).max() < 1e-12
    U = g.get_state(0).cpu().numpy()
    assert np.abs(U.conj().T @ U - np.eye(L // 2)).max() < 1e-12
    assert not g.failed(0)


@pytest.mark.parametrize("P_shards", [2, 4, 8])
def test_row_sharded_chunked_propagate_matches_single_gemm(P, P_shards, monkeypatch):
    """The sharded dense propagate as P ring-ordered K-chunk GEMMs (the schedule that overlaps
    the per-distance exchange with compute in NCCL mode, SURVEY §8(e) "fusion with the
    collective") equals the allgather + one L-deep GEMM (TRAJ_SHARD_OVERLAP=0) to rounding,
    and both equal the oracle."""
    L = 512
    monkeypatch.setenv("TRAJ_SHARD_OVERLAP", "0")
    a = P.Trajectories(L, 1, "projective", [2.0], seed=21, shard_size=P_shards)
    monkeypatch.setenv("TRAJ_SHARD_OVERLAP", "1")
    b = P.Trajectories(L, 1, "projective", [2.0], seed=21, shard_size=P_shards)
    K = lattice.propagator_lattice(L, 1, 1.0, 0.05)
    o = OracleTrajectory(L, 1, "projective", 2.0, 0.05, seed=21, traj=0, K=K)
    for s in range(6):
        a.step(1)
        b.step(1)
        o.step(1)
        assert a.last_clicks(0) == b.last_clicks(0)
    ca, cb = a.correlation(0).cpu().numpy(), b.correlation(0).cpu().numpy()
    assert np.abs(ca - cb).max() < 1e-13
    assert np.abs(cb - o.correlation()).max() < C_TOL
    a.close()
    b.close()


@pytest.mark.parametrize("P_shards", [2, 4, 8])
def test_row_sharded_distributed_cholesky_matches_replicated(P, P_shards, monkeypatch):
    """The N x N Cholesky of the row-sharded CholeskyQR with its recursion levels split into row
    slices over the ranks (every level >= 64 here; the emulation computes each rank's slice in
    turn, exercising the slice offsets of the triangular / upper-tile GEMMs; at P = 8 some slices
    round to empty): the same state as the replicated factorisation, and the oracle's."""
    L = 512
    monkeypatch.setenv("TRAJ_DIST_CHOL_MIN", "0")
    a = P.Trajectories(L, 1, "projective", [1.5], seed=33, shard_size=P_shards)
    monkeypatch.setenv("TRAJ_DIST_CHOL_MIN", "64")
    b = P.Trajectories(L, 1, "projective", [1.5], seed=33, shard_size=P_shards)
    K = lattice.propagator_lattice(L, 1, 1.0, 0.05)
    o = OracleTrajectory(L, 1, "projective", 1.5, 0.05, seed=33, traj=0, K=K)
    for s in range(8):
        a.step(1)
        b.step(1)
        o.step(1)
        assert a.last_clicks(0) == b.last_clicks(0)
    ca, cb = a.correlation(0).cpu().numpy(), b.correlation(0).cpu().numpy()
    assert np.abs(ca - cb).max() < 1e-12
    assert np.abs(cb - o.correlation()).max() < C_TOL
    U = b.get_state(0).cpu().numpy()
    assert np.abs(U.conj().T @ U - np.eye(L // 2)).max() < 1e-12
    a.close()
    b.close()


@pytest.mark.parametrize("Lx,Ly,protocol,gams", [(300, 1, "projective", [2.0]), (12, 10, "homodyne", [1.0, 3.0]),
                                                  (260, 1, "projective", [1.0, 2.5, 0.3])])
def test_planar_propagator_matches_interleaved(P, Lx, Ly, protocol, gams, monkeypatch):
    """The planar 3M paths (K U as three real products; CholeskyQR's Grams and TRMMs likewise, with
    the plane-major batching of several trajectories) against the interleaved complex 3M kernels
    and the oracle, same trajectories.  TRAJ_PLANAR_MIN_N=0 turns the planar paths on at these
    small sizes."""
    monkeypatch.setenv("TRAJ_PLANAR_MIN_N", "0")
    monkeypatch.setenv("TRAJ_OZAKI", "0")
    monkeypatch.setenv("TRAJ_PLANAR_KU", "0")
    monkeypatch.setenv("TRAJ_PLANAR_CQR", "0")
    a = P.Trajectories(Lx, Ly, protocol, gams, seed=41)
    monkeypatch.setenv("TRAJ_PLANAR_KU", "1")
    monkeypatch.setenv("TRAJ_PLANAR_CQR", "1")
    b = P.Trajectories(Lx, Ly, protocol, gams, seed=41)
    K = lattice.propagator_lattice(Lx, Ly, 1.0, 0.05)
    orc = [OracleTrajectory(Lx, Ly, protocol, g, 0.05, seed=41, traj=t, K=K) for t, g in enumerate(gams)]
    for s in range(12):
        a.step(1)
        b.step(1)
        for t, o in enumerate(orc):
            o.step(1)
            if protocol == "projective":
                assert a.last_clicks(t) == b.last_clicks(t)
    for t, o in enumerate(orc):
        ca, cb = a.correlation(t).cpu().numpy(), b.correlation(t).cpu().numpy()
        assert np.abs(ca - cb).max() < 1e-12
        assert np.abs(cb - o.correlation()).max() < C_TOL
    a.close()
    b.close()


@pytest.mark.parametrize("planar", [False, True])
def test_row_sharded_nccl_single_rank(P, planar, monkeypatch):
    """The NCCL code path of the sharded step with a one-rank communicator (the only
    configuration one GPU allows): same result as the unsharded handle.  planar: the planar
    Gram with its packed, pipelined allreduce by 64-column panels (ragged last panel)."""
    L = 232 if planar else 128
    if planar:
        monkeypatch.setenv("TRAJ_PLANAR_MIN_N", "0")
        monkeypatch.setenv("TRAJ_OZAKI", "0")
        monkeypatch.setenv("TRAJ_GRAM_PANEL", "64")
    uid = P.traj_nccl_unique_id()
    a = P.Trajectories(L, 1, "projective", [3.0], seed=5, shard_size=1, shard_rank=0, nccl_id=uid)
    b = P.Trajectories(L, 1, "projective", [3.0], seed=5)
    a.step(10)
    b.step(10)
    assert a.last_clicks(0) == b.last_clicks(0)
    assert np.abs(a.correlation(0).cpu().numpy() - b.correlation(0).cpu().numpy()).max() < 1e-12
    assert abs(a.entropy(np.arange(64))[0] - b.entropy(np.arange(64))[0]) < 1e-10
    U = a.get_state(0).cpu().numpy()
    assert np.abs(U.conj().T @ U - np.eye(L // 2)).max() < 1e-12
    a.close()


@pytest.mark.parametrize("shards", [1, 4])
def test_density_correlation_and_particle_covariance(P, shards):
    """NEXT-3: C(r) of Eq. (2) and G_AB of Eq. (5) against the oracle (blocks of U U^dag on the
    GEMM, deterministic binning); also through the row-sharded handle."""
    L = 320
    g = P.Trajectories(L, 1, "homodyne", [0.7], seed=2, shard_size=shards)
    K = lattice.propagator_lattice(L, 1, 1.0, 0.05)
    o = OracleTrajectory(L, 1, "homodyne", 0.7, 0.05, seed=2, traj=0, K=K)
    g.step(25)
    o.step(25)
    Cr = g.density_correlation(0)
    want = gaussian.density_correlation(o.U)
    assert np.isnan(Cr[0])
    assert np.abs(Cr[1:] - want[1:]).max() < 1e-13
    A, B = np.arange(0, 80), np.arange(160, 240)
    G = g.particle_covariance(A, B)[0]
    assert G == pytest.approx(gaussian.particle_covariance(o.U, A, B), rel=1e-11, abs=1e-13)


def test_particle_covariance_2d_batch(P):
    """G_AB between the c4/c5 strips on a 2d torus, batched trajectories."""
    A, B = workloads.strips_2d(12, 12)
    g = P.Trajectories(12, 12, "projective", [2.86, 5.72], seed=1)
    K = lattice.propagator_lattice(12, 12, 1.0, 0.05)
    orc = [OracleTrajectory(12, 12, "projective", gm, 0.05, seed=1, traj=t, K=K) for t, gm in enumerate([2.86, 5.72])]
    g.step(15)
    for o in orc:
        o.step(15)
    G = g.particle_covariance(A, B)
    for t, o in enumerate(orc):
        assert G[t] == pytest.approx(gaussian.particle_covariance(o.U, A, B), rel=1e-11, abs=1e-13)


@pytest.mark.parametrize("Lx,Ly,protocol,gam", [(240, 1, "homodyne", 1.0), (200, 1, "projective", 3.0),
                                                (14, 10, "homodyne", 2.0), (12, 12, "projective", 2.86),
                                                (15, 10, "homodyne", 2.0)])
def test_banded_propagator_matches_dense_oracle(P, Lx, Ly, protocol, gam):
    """NEXT-1: banded circulant passes (1d) / K_y (x) K_x as two passes (2d) against the oracle's
    dense exact K: the dropped Bessel tail is below 1e-18, so the lockstep bar is unchanged.  An
    odd axis (15) has taps that are not purely real / imaginary: the four-FMA kernel there."""
    lockstep_kw = dict(seed=6)
    gpu = P.Trajectories(Lx, Ly, protocol, [gam, gam / 2], propagator="banded", **lockstep_kw)
    K = lattice.propagator_lattice(Lx, Ly, 1.0, 0.05)
    orc = [OracleTrajectory(Lx, Ly, protocol, g, 0.05, seed=6, traj=t, K=K) for t, g in enumerate([gam, gam / 2])]
    A = np.arange(Lx * Ly // 2)
    for s in range(30):
        gpu.step(1)
        for o in orc:
            o.step(1)
    S = gpu.entropy(A)
    for t, o in enumerate(orc):
        assert np.abs(gpu.correlation(t).cpu().numpy() - o.correlation()).max() < C_TOL
        assert abs(S[t] - o.entropy(A)) < S_TOL


def test_banded_free_evolution_closed_form_full_c3(P):
    """configs[2] size with the banded propagator: finite-L closed form after 40 steps."""
    L, steps, dt = 16384, 40, 0.05
    g = P.Trajectories(L, 1, "projective", [0.0], dt=dt, propagator="banded")
    g.step(steps)
    n = g.occupations()[0].cpu().numpy()
    m = np.arange(L)
    want = 0.5 + 0.5 * (-1.0) ** m * np.mean(np.cos(4 * steps * dt * np.cos(2 * np.pi * m / L)))
    assert np.abs(n - want).max() < 1e-12


@pytest.mark.parametrize("Lx,Ly", [(200, 1), (10, 8)])
def test_rk4_qsd_protocol_matches_oracle(P, Lx, Ly):
    """NEXT-2: the paper-literal QSD integrator (RK4 on the Eq. A3 generator) in lockstep
    with the oracle's literal RK4 stages (the GPU evaluates the same polynomial in Horner form)."""
    A = np.arange(Lx * Ly // 2)
    lockstep(P, Lx, Ly, "homodyne_rk4", [0.3, 2.0], 60, 20, [A], seed=12)


@pytest.mark.parametrize("Lx,Ly,gam,orth", [(64, 1, 3.0, "cqr2"), (96, 1, 0.5, "cqr2"), (8, 6, 4.0, "cqr2"),
                                             (100, 1, 2.0, "lowrank"), (8, 6, 4.0, "lowrank")])
def test_event_driven_pm_matches_oracle(P, Lx, Ly, gam, orth):
    """NEXT-4: the paper-literal event-driven PM (Poisson waiting times, one site per event,
    Eq. A1/A2 on the L x L matrix in the oracle) against the GPU's orbital form (banded K(tau)
    stencils and exact rank-1 updates; 1d: the row-blocked kernel, L = 100 leaves a ragged last
    block), with the same Philox event stream.  orth = "lowrank": the window's CholeskyQR runs
    only when the orthonormality probe sees drift."""
    from oracle.pm_events import EventPM
    g = P.Trajectories(Lx, Ly, "projective_events", [gam, gam * 1.5], seed=3, orthonormalizer=orth)
    orc = [EventPM(Lx, Ly, gm, 0.05, seed=3, traj=t) for t, gm in enumerate([gam, gam * 1.5])]
    A = np.arange(Lx * Ly // 2)
    events = 0
    for s in range(1, 41):
        g.step(1)
        for t, o in enumerate(orc):
            n0 = len(o.log)
            o.step(1)
            nev, nocc = g.last_clicks(t)
            assert nev == len(o.log) - n0
            assert nocc == sum(1 for e in o.log[n0:] if e[3])
            events += nev
        if s % 10 == 0:
            S = g.entropy(A)
            for t, o in enumerate(orc):
                assert np.abs(g.correlation(t).cpu().numpy() - o.correlation()).max() < C_TOL
                assert abs(S[t] - o.entropy(A)) < S_TOL
    assert events > 50


@pytest.mark.parametrize("Lx,Ly,gam,steps,min_events", [(12, 10, 3.0, 20, 100), (28, 27, 10.0, 2, 200)])
def test_event_driven_pm_2d_separable_pass_matches_product_taps_and_oracle(P, monkeypatch, Lx, Ly, gam, steps,
                                                                           min_events):
    """NEXT-4 on a 2d lattice: the separable pass (x-axis taps into a scratch copy, then y-axis taps
    with the rank-1 term; the default) and the (2w+1)^2 product taps in one kernel
    (TRAJ_EV_SEPARABLE=0) give the same trajectory, and both follow the oracle's literal L x L
    algorithm on a non-square lattice.  12 x 10: both halves one CTA per row (the rings
    are too short for the row-blocked kernel); 28 x 27 at a high event rate (short waiting times,
    narrow bands): both halves on the row-blocked ring kernel, ragged last row blocks on both axes."""
    from oracle.pm_events import EventPM
    A = np.arange(Lx * Ly // 2)
    res = {}
    for sep in ("1", "0"):
        monkeypatch.setenv("TRAJ_EV_SEPARABLE", sep)
        g = P.Trajectories(Lx, Ly, "projective_events", [gam], seed=5)
        o = EventPM(Lx, Ly, gam, 0.05, seed=5, traj=0)
        events = 0
        for s in range(steps):
            g.step(1)
            n0 = len(o.log)
            o.step(1)
            nev, nocc = g.last_clicks(0)
            assert nev == len(o.log) - n0
            assert nocc == sum(1 for e in o.log[n0:] if e[3])
            events += nev
        assert events > min_events
        C = g.correlation(0).cpu().numpy()
        assert np.abs(C - o.correlation()).max() < C_TOL
        assert abs(g.entropy(A)[0] - o.entropy(A)) < S_TOL
        res[sep] = C
    assert np.abs(res["1"] - res["0"]).max() < 1e-12


@pytest.mark.parametrize("Lx,Ly,P_shards,protocol", [(256, 1, 4, "projective"), (240, 1, 2, "homodyne"),
                                                     (12, 12, 3, "projective"), (10, 8, 2, "homodyne")])
def test_row_sharded_banded_halo_matches_oracle(P, Lx, Ly, P_shards, protocol):
    """NEXT-1 with sharding: the halo exchange (W rows in 1d, W*Lx rows for the 2d y pass)
    replaces the allgather; lockstep with the oracle's dense K."""
    gam = 3.0 if protocol == "projective" else 1.0
    g = P.Trajectories(Lx, Ly, protocol, [gam], seed=21, shard_size=P_shards, propagator="banded")
    K = lattice.propagator_lattice(Lx, Ly, 1.0, 0.05)
    o = OracleTrajectory(Lx, Ly, protocol, gam, 0.05, seed=21, traj=0, K=K)
    A = np.arange(Lx * Ly // 2)
    for s in range(20):
        g.step(1)
        o.step(1)
    assert np.abs(g.correlation(0).cpu().numpy() - o.correlation()).max() < C_TOL
    assert abs(g.entropy(A)[0] - o.entropy(A)) < S_TOL


def test_row_sharded_banded_nccl_single_rank(P):
    """Halo exchange through NCCL send/recv with a one-rank communicator (neighbours = self)."""
    uid = P.traj_nccl_unique_id()
    a = P.Trajectories(128, 1, "homodyne", [1.0], seed=5, shard_size=1, nccl_id=uid, propagator="banded")
    b = P.Trajectories(128, 1, "homodyne", [1.0], seed=5)
    a.step(10)
    b.step(10)
    assert np.abs(a.correlation(0).cpu().numpy() - b.correlation(0).cpu().numpy()).max() < 1e-12
    a.close()


@pytest.mark.parametrize("protocol,gam", [("homodyne", 0.5), ("projective", 1.0)])
def test_long_run_trajectory_averaged_entropy(P, protocol, gam):
    """North star: trajectory-averaged S_A within statistical error over long runs (here 600
    steps, t = 30, 24 trajectories at L = 128): Welch-type |mean_gpu - mean_oracle| < 3 sigma at
    every sample time.  The trajectories also stay individually close (contraction of
    perturbations), which the looser ensemble bound does not rely on."""
    L, T, steps, every = 128, 24, 600, 100
    A = np.arange(L // 2)
    g = P.Trajectories(L, 1, protocol, [gam] * T, seed=31)
    K = lattice.propagator_lattice(L, 1, 1.0, 0.05)
    orc = [OracleTrajectory(L, 1, protocol, gam, 0.05, seed=31, traj=t, K=K) for t in range(T)]
    for s in range(every, steps + 1, every):
        g.step(every)
        for o in orc:
            o.step(every)
        sg = g.entropy(A)
        so = np.array([o.entropy(A) for o in orc])
        sigma = np.sqrt(sg.var(ddof=1) / T + so.var(ddof=1) / T)
        assert abs(sg.mean() - so.mean()) < 3 * sigma + 1e-12
        assert np.abs(sg - so).max() < 1e-6


def test_projective_lowrank_first_gram_matches_measured(P):
    """The projective step forms CholeskyQR2's first Gram as I - V^dag V (V: the rows zeroed by
    the empty outcomes; U is orthonormal before zeroing) instead of U'^dag U'; the second pass
    measures the Gram.  Same state as with the measured first Gram (TRAJ_LOWRANK_GRAM=0)."""
    import os
    args = (300, 1, "projective", [3.0, 0.5])
    a = P.Trajectories(*args, seed=17)
    os.environ["TRAJ_LOWRANK_GRAM"] = "0"
    try:
        b = P.Trajectories(*args, seed=17)
    finally:
        del os.environ["TRAJ_LOWRANK_GRAM"]
    a.step(40)
    b.step(40)
    for t in range(2):
        assert a.last_clicks(t) == b.last_clicks(t)
        assert np.abs(a.correlation(t).cpu().numpy() - b.correlation(t).cpu().numpy()).max() < 1e-12
        U = a.get_state(t).cpu().numpy()
        assert np.abs(U.conj().T @ U - np.eye(150)).max() < 1e-13


@pytest.mark.parametrize("Lx,Ly,gams", [(300, 1, [3.0, 0.5]), (10, 10, [2.86, 5.72]), (400, 1, [10.0])])
def test_lowrank_projective_orthonormalizer_matches_oracle(P, Lx, Ly, gams):
    """NEXT-1 option: the projective step orthonormalised at low rank (Newton-Schulz on the
    k0 x k0 block, two O(L N k0) GEMMs), certified each step by the orthonormality probe with a
    measured CholeskyQR refinement above its tolerance, in lockstep with the oracle
    (Householder QR)."""
    g = P.Trajectories(Lx, Ly, "projective", gams, seed=23, orthonormalizer="lowrank")
    K = lattice.propagator_lattice(Lx, Ly, 1.0, 0.05)
    orc = [OracleTrajectory(Lx, Ly, "projective", gm, 0.05, seed=23, traj=t, K=K) for t, gm in enumerate(gams)]
    A = np.arange(Lx * Ly // 2)
    for s in range(25):
        g.step(1)
        for t, o in enumerate(orc):
            o.step(1)
            assert g.last_clicks(t) == (o.last_clicks[0].size, int(o.last_clicks[1].sum()))
    S = g.entropy(A)
    for t, o in enumerate(orc):
        assert np.abs(g.correlation(t).cpu().numpy() - o.correlation()).max() < C_TOL
        assert abs(S[t] - o.entropy(A)) < S_TOL
        U = g.get_state(t).cpu().numpy()
        assert np.abs(U.conj().T @ U - np.eye(U.shape[1])).max() < 1e-13


def _random_orthonormal(L, N, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((L, N)) + 1j * rng.standard_normal((L, N)))
    return Q


def test_probe_orthonormality_estimates_gram_deviation(P):
    """The orthonormality certificate (probe.cu): est = sqrt(mean_j ||U^dag U x_j - x_j||^2) for 4
    unit-modulus random probes estimates ||E||_F, E = U^dag U - I (Hutchinson, E[x x^dag] = I).
    Pinned against the exact E from NumPy: an orthonormal U reads at rounding level; a diffuse
    E = 2 eps H + eps^2 H^2 within the estimator's spread (relative std ~ sqrt(2/(4N)) ~ 6%);
    an error confined to one entry pair exactly (|x_k| = 1)."""
    import torch
    L, N = 256, 128
    g = P.Trajectories(L, 1, "homodyne", [0.5, 0.5, 0.5], seed=3)
    Q = _random_orthonormal(L, N, 1)
    rng = np.random.default_rng(2)
    H = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))
    H = (H + H.conj().T) / 2
    U1 = Q @ (np.eye(N) + 1e-7 * H)
    B = np.eye(N, dtype=complex)
    B[5, 77] += 3e-7 - 2e-7j
    U2 = Q @ B
    for t, U in enumerate((Q, U1, U2)):
        g.set_state(t, torch.from_numpy(np.ascontiguousarray(U)).cuda())
    est = g.probe_orthonormality()
    exact = [np.linalg.norm(U.conj().T @ U - np.eye(N)) for U in (Q, U1, U2)]
    assert est[0] < 1e-13
    assert 0.7 < est[1] / exact[1] < 1.3
    assert abs(est[2] / exact[2] - 1) < 1e-4
    g.close()


def test_lowrank_probe_gates_refinement(P, monkeypatch):
    """With the low-rank orthonormaliser the measured CholeskyQR pass runs only when the probe
    sees ||U^dag U - I||_F above TRAJ_LOWRANK_TOL: over 300 steps the state stays orthonormal to
    the tolerance, the oracle-lockstep C agrees, a tight tolerance refines more often than a
    loose one, and TRAJ_LOWRANK_TOL=0 refines every step without probing."""
    L, gam, steps = 400, 2.0, 300
    K = lattice.propagator_lattice(L, 1, 1.0, 0.05)
    o = OracleTrajectory(L, 1, "projective", gam, 0.05, seed=31, traj=0, K=K)
    res = {}
    for tol in ("5e-13", "5e-14", "0"):
        monkeypatch.setenv("TRAJ_LOWRANK_TOL", tol)
        g = P.Trajectories(L, 1, "projective", [gam], seed=31, orthonormalizer="lowrank")
        g.step(steps)
        U = g.get_state(0).cpu().numpy()
        E = U.conj().T @ U - np.eye(L // 2)
        res[tol] = (g.lowrank_stats(), np.linalg.norm(E), g.correlation(0).cpu().numpy())
        g.close()
    o.step(steps)
    for tol, (st, nE, C) in res.items():
        assert nE < max(float(tol), 5e-14) * 3, (tol, nE)
        assert np.abs(C - o.correlation()).max() < C_TOL
        assert st["fallbacks"] == 0
    assert res["0"][0]["probes"] == 0
    assert res["5e-13"][0]["probes"] >= steps // 2
    assert res["5e-13"][0]["refinements"] < res["5e-14"][0]["refinements"]


@pytest.mark.parametrize("orth", ["cqr2", "lowrank"])
def test_projective_l4096_lockstep(P, orth):
    """L = 4096 (N = 2048): large enough for the split-K skinny products of the projective step
    (U W, and U' V^dag in the low-rank mode, K = N as one batch-2 launch) and for the planar
    paths at their default threshold; three steps in lockstep with the oracle."""
    L, gam = 4096, 0.5
    g = P.Trajectories(L, 1, "projective", [gam], seed=17, orthonormalizer=orth)
    K = lattice.propagator_lattice(L, 1, 1.0, 0.05)
    o = OracleTrajectory(L, 1, "projective", gam, 0.05, seed=17, traj=0, K=K)
    for s in range(3):
        g.step(1)
        o.step(1)
        assert g.last_clicks(0) == (o.last_clicks[0].size, int(o.last_clicks[1].sum()))
    assert np.abs(g.correlation(0).cpu().numpy() - o.correlation()).max() < C_TOL
    A = np.arange(L // 2)
    assert abs(g.entropy(A)[0] - o.entropy(A)) < S_TOL


@pytest.mark.parametrize("Lx,Ly,protocol,gams", [(64, 1, "projective", [0.5, 0.3, 2.0]), (8, 8, "projective", [2.86]),
                                                  (12, 8, "homodyne", [0.5, 3.0]), (50, 1, "homodyne", [1.0]),
                                                  (10, 1, "projective", [20.0, 20.0]), (2, 1, "projective", [5.0]),
                                                  (104, 1, "projective", [4.0]), (10, 10, "projective", [5.72])])
def test_small_step_matches_general_path_and_oracle(P, Lx, Ly, protocol, gams, monkeypatch):
    """The fused small-lattice step (small_step.cu: one CTA per trajectory, U in shared memory)
    against the general multi-kernel path (TRAJ_SMALL_STEP=0) and the oracle on the same Philox
    streams: identical click lists and outcomes, C within the north-star bar.  gamma dt = 1
    (every site clicks) puts C_SS in global memory; L = 2 is the smallest lattice, L = 104 the largest
    1d ring whose state fits one CTA's shared memory."""
    monkeypatch.setenv("TRAJ_SMALL_STEP", "0")
    a = P.Trajectories(Lx, Ly, protocol, gams, seed=23, traj_base=3)
    monkeypatch.setenv("TRAJ_SMALL_STEP", "1")
    b = P.Trajectories(Lx, Ly, protocol, gams, seed=23, traj_base=3)
    K = lattice.propagator_lattice(Lx, Ly, 1.0, 0.05)
    orc = [OracleTrajectory(Lx, Ly, protocol, g, 0.05, seed=23, traj=3 + t, K=K) for t, g in enumerate(gams)]
    n0 = P.traj_kernel_launches()
    b.step(1)
    assert P.traj_kernel_launches() - n0 == 1          # the fused path ran: one launch per call
    a.step(1)
    for t, o in enumerate(orc):
        o.step(1)
    for s in range(1, 25):
        if protocol == "projective":
            for t, o in enumerate(orc):
                S_, occ = o.last_clicks
                assert a.last_clicks(t) == b.last_clicks(t) == (S_.size, int(occ.sum())), (s, t)
        a.step(1)
        b.step(1)
        for o in orc:
            o.step(1)
    for t, o in enumerate(orc):
        assert not b.failed(t)
        ca, cb = a.correlation(t).cpu().numpy(), b.correlation(t).cpu().numpy()
        assert np.abs(ca - cb).max() < C_TOL
        assert np.abs(cb - o.correlation()).max() < C_TOL
        U = b.get_state(t).cpu().numpy()
        assert np.abs(U.conj().T @ U - np.eye(U.shape[1])).max() < 1e-13
    A = np.arange(Lx * Ly // 2)
    assert np.abs(b.entropy(A) - np.array([o.entropy(A) for o in orc])).max() < S_TOL
    a.close()
    b.close()


def test_small_step_multi_step_launch_is_step_by_step(P):
    """traj_step(n) runs n steps inside one launch: bit-identical to n calls of one step (same
    kernel, same counters), and the click counts reported are those of the last step."""
    a = P.Trajectories(64, 1, "projective", [0.5, 1.5], seed=9)
    b = P.Trajectories(64, 1, "projective", [0.5, 1.5], seed=9)
    n0 = P.traj_kernel_launches()
    a.step(40)
    assert P.traj_kernel_launches() - n0 == 1
    for _ in range(40):
        b.step(1)
    for t in range(2):
        assert a.last_clicks(t) == b.last_clicks(t)
        assert np.array_equal(a.get_state(t).cpu().numpy(), b.get_state(t).cpu().numpy())
    assert a.step_index == b.step_index == 40
    a.close()
    b.close()


def test_small_step_first_order_second_pass_and_fallback(P, monkeypatch):
    """The fused step's CholeskyQR2 second pass uses the first-order R2^-1 (the general path's rule
    and threshold): strong homodyne reweighting (gamma dt = 5, kappa up to ~3e4) gives the same
    states as the full second factorisation (TRAJ_CQR2_FULL=1), the general path and the oracle;
    an ill-conditioned state (kappa ~ 1e5: pass 1 leaves |E| ~ 1e-6) must fall back to the full
    factorisation, counted by traj_cqr2_fallbacks."""
    import torch
    args = (32, 1, "homodyne", [100.0])
    monkeypatch.setenv("TRAJ_SMALL_STEP", "0")
    a = P.Trajectories(*args, seed=6)
    monkeypatch.setenv("TRAJ_SMALL_STEP", "1")
    b = P.Trajectories(*args, seed=6)
    monkeypatch.setenv("TRAJ_CQR2_FULL", "1")
    c = P.Trajectories(*args, seed=6)
    monkeypatch.delenv("TRAJ_CQR2_FULL")
    K = lattice.propagator_lattice(32, 1, 1.0, 0.05)
    o = OracleTrajectory(32, 1, "homodyne", 100.0, 0.05, seed=6, traj=0, K=K)
    for _ in range(20):
        a.step(1)
        b.step(1)
        c.step(1)
        o.step(1)
    cb = b.correlation(0).cpu().numpy()
    assert np.abs(cb - a.correlation(0).cpu().numpy()).max() < C_TOL
    assert np.abs(cb - c.correlation(0).cpu().numpy()).max() < 1e-12
    assert np.abs(cb - o.correlation()).max() < C_TOL
    # gamma = 0: one step is K U, then CholeskyQR2 of the ill-conditioned K U
    L, N = 32, 16
    U = workloads.random_matrix(L, N, 3)
    U[:, 1] = U[:, 0] + 1e-5 * U[:, 1]
    d = P.Trajectories(L, 1, "homodyne", [0.0])
    d.set_state(0, torch.from_numpy(U).cuda())
    n0 = d.cqr2_fallbacks()
    d.step(1)
    assert d.cqr2_fallbacks() - n0 == 1
    Ud = d.get_state(0).cpu().numpy()
    assert np.abs(Ud.conj().T @ Ud - np.eye(N)).max() < 1e-12
    ref = gaussian.correlation(gaussian.orthonormalize(K @ U))
    assert np.abs(d.correlation(0).cpu().numpy() - ref).max() < 1e-9
    for h in (a, b, c, d):
        h.close()


def test_small_step_failed_trajectory_is_flagged_and_frozen(P):
    """A rank-deficient state makes the fused step's Cholesky break down: that trajectory is
    flagged (traj_failed) and stops evolving, the other trajectories of the batch are unaffected
    and still match the oracle."""
    import torch
    L = 32
    g = P.Trajectories(L, 1, "homodyne", [0.5, 0.5], seed=8)
    U = workloads.random_matrix(L, L // 2, 5)
    U[:, 1] = U[:, 0]                         # exactly rank deficient
    g.set_state(0, torch.from_numpy(U).cuda())
    g.step(3)
    assert g.failed(0) and not g.failed(1)
    U0 = g.get_state(0).cpu().numpy()
    g.step(2)
    assert np.array_equal(g.get_state(0).cpu().numpy(), U0)   # frozen
    K = lattice.propagator_lattice(L, 1, 1.0, 0.05)
    o = OracleTrajectory(L, 1, "homodyne", 0.5, 0.05, seed=8, traj=1, K=K)
    o.step(5)
    assert np.abs(g.correlation(1).cpu().numpy() - o.correlation()).max() < C_TOL
    g.close()


def test_small_step_size_boundary(P):
    """L = 104 (N = 52) still fits the fused step (one launch per call); L = 106 does not and runs
    the general multi-kernel path."""
    a = P.Trajectories(104, 1, "homodyne", [0.5])
    b = P.Trajectories(106, 1, "homodyne", [0.5])
    n0 = P.traj_kernel_launches()
    a.step(3)
    n1 = P.traj_kernel_launches()
    b.step(3)
    n2 = P.traj_kernel_launches()
    assert n1 - n0 == 1 and n2 - n1 > 3
    a.close()
    b.close()


def test_event_pass_alternating_taps_match_general(P, monkeypatch):
    """The 1d event pass with the two-FMA taps (K(tau)'s taps alternate real / imaginary on the
    bipartite ring) against the general four-FMA taps (TRAJ_EV_ALT_TAPS=0), same event stream:
    identical event outcomes and states equal to rounding."""
    a = P.Trajectories(200, 1, "projective_events", [2.0], seed=13)
    b = P.Trajectories(200, 1, "projective_events", [2.0], seed=13)
    for _ in range(20):
        monkeypatch.setenv("TRAJ_EV_ALT_TAPS", "0")
        a.step(1)
        monkeypatch.setenv("TRAJ_EV_ALT_TAPS", "1")
        b.step(1)
        assert a.last_clicks(0) == b.last_clicks(0)
    assert np.abs(a.get_state(0).cpu().numpy() - b.get_state(0).cpu().numpy()).max() < 1e-13
    a.close()
    b.close()


def test_banded_alternating_taps_match_general(P, monkeypatch):
    """The banded stencil with two-FMA taps (even ring: taps alternate real / imaginary) against the
    four-FMA taps (TRAJ_BANDED_ALT_TAPS=0): the same trajectory to rounding."""
    a = P.Trajectories(256, 1, "homodyne", [1.0], propagator="banded", seed=21)
    b = P.Trajectories(256, 1, "homodyne", [1.0], propagator="banded", seed=21)
    for _ in range(10):
        monkeypatch.setenv("TRAJ_BANDED_ALT_TAPS", "0")
        a.step(1)
        monkeypatch.delenv("TRAJ_BANDED_ALT_TAPS")
        b.step(1)
    assert np.abs(a.get_state(0).cpu().numpy() - b.get_state(0).cpu().numpy()).max() < 1e-13
    a.close()
    b.close()


def test_phase_times_attribute_the_fused_step(P):
    """traj_phase_times: the fused small-lattice step records its whole time and its one launch per
    call under "fused"; the general path leaves "fused" at zero."""
    a = P.Trajectories(64, 1, "projective", [0.5, 0.5], seed=1)
    b = P.Trajectories(200, 1, "projective", [0.5], seed=1)
    for h in (a, b):
        h.profile(True)
        h.step(5)
    pa, pb = a.phase_times(), b.phase_times()
    assert pa["fused"][0] > 0 and pa["fused"][1] == 1
    assert all(pa[k] == (0.0, 0) for k in pa if k != "fused")
    assert pb["fused"] == (0.0, 0) and pb["propagate"][0] > 0 and pb["gram"][1] > 0
    a.close()
    b.close()
