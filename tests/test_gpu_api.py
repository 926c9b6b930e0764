"""C-ABI behaviour on the GPU: checkpoint/resume, determinism, failure isolation, domain errors
(SURVEY §5 and §8(b) conventions)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("protocol", ["projective", "homodyne", "homodyne_rk4", "projective_events"])
def test_checkpoint_resume_is_exact(P, protocol):
    """(state, step) is a complete checkpoint: counter-based Philox makes the resumed run
    bitwise identical to the uninterrupted one."""
    a = P.Trajectories(96, 1, protocol, [2.0, 0.5], seed=7, traj_base=3)
    a.step(30)
    b = P.Trajectories(96, 1, protocol, [2.0, 0.5], seed=7, traj_base=3)
    b.step(18)
    states = [b.get_state(t).clone() for t in range(2)]
    step = b.step_index
    b.close()
    c = P.Trajectories(96, 1, protocol, [2.0, 0.5], seed=7, traj_base=3)
    for t in range(2):
        c.set_state(t, states[t])
    c.step_index = step
    c.step(12)
    for t in range(2):
        assert np.array_equal(a.get_state(t).cpu().numpy(), c.get_state(t).cpu().numpy())


def test_determinism(P):
    """Same seed, same configuration: bitwise identical correlation matrices and entropies."""
    runs = []
    for _ in range(2):
        g = P.Trajectories(10, 10, "projective", [2.86, 5.72], seed=11)
        g.step(20)
        runs.append((g.correlation(0).cpu().numpy(), g.entropy(np.arange(50))))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])


def test_failure_is_isolated(P):
    """A rank-deficient state breaks the Cholesky of its own trajectory only: it is flagged,
    its entropy is NaN, and the other trajectory of the batch is untouched."""
    import torch
    g = P.Trajectories(64, 1, "homodyne", [1.0, 1.0], seed=2)
    ref = P.Trajectories(64, 1, "homodyne", [1.0, 1.0], seed=2)
    U = g.get_state(0).clone()
    U[:, 3] = 0.0                      # a vanishing orbital: G singular
    g.set_state(0, U)
    g.step(3)
    ref.step(3)
    assert g.failed(0) and not g.failed(1)
    S = g.entropy(np.arange(32))
    assert np.isnan(S[0]) and np.isfinite(S[1])
    assert np.abs(g.correlation(1).cpu().numpy() - ref.correlation(1).cpu().numpy()).max() == 0.0


def test_domain_errors_keep_the_handle_usable(P):
    g = P.Trajectories(32, 1, "projective", [1.0], seed=0)
    for bad in (lambda: g.entropy([0, 0, 1]),                      # duplicate site
                lambda: g.entropy([40]),                           # outside the lattice
                lambda: g.mutual_info([0, 1], [1, 2]),             # overlapping regions
                lambda: g.particle_covariance([0, 1], [1, 2])):
        with pytest.raises(P.TrajError) as e:
            bad()
        assert e.value.status == 6                                 # TRAJ_EDOMAIN
    with pytest.raises(P.TrajError) as e:
        g.correlation_rows(3, 0, 4)                                # trajectory index out of range
    assert e.value.status == 1
    g.step(2)                                                      # still usable
    assert np.isfinite(g.entropy(np.arange(16))).all()
    assert g.entropy([])[0] == 0.0


def test_2d_density_correlation_is_a_domain_error(P):
    g = P.Trajectories(6, 6, "homodyne", [1.0])
    with pytest.raises(P.TrajError) as e:
        g.density_correlation(0)
    assert e.value.status == 6


@pytest.mark.parametrize("protocol,shards", [("projective", 1), ("homodyne", 1), ("projective", 2),
                                             ("homodyne_rk4", 1)])
def test_traj_step_is_asynchronous(P, protocol, shards):
    """calls are stream-ordered and asynchronous unless they return host values.
    traj_step sizes the projective launches from the host's own counter-based click counts and
    decides CholeskyQR2's second pass on the device, so it returns while the GPU is still busy
    (the stream reports work pending) -- and the result is unchanged (checked against a run that
    synchronises after every step)."""
    import time
    import torch
    L = 4096
    a = P.Trajectories(L, 1, protocol, [0.6], seed=11, shard_size=shards)
    a.step(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.step(3)
    host_ms = 1e3 * (time.perf_counter() - t0)
    pending = not a.stream.query()
    torch.cuda.synchronize()
    assert pending, f"traj_step returned after the GPU finished ({host_ms:.2f} ms on the host)"
    b = P.Trajectories(L, 1, protocol, [0.6], seed=11, shard_size=shards)
    for _ in range(4):
        b.step(1)
        torch.cuda.synchronize()
    assert a.last_clicks(0) == b.last_clicks(0)
    assert np.abs(a.get_state(0).cpu().numpy() - b.get_state(0).cpu().numpy()).max() == 0.0
    a.close()
    b.close()
