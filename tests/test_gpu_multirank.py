"""Multi-rank NCCL execution of the row-sharded step and its failure detection.

- With >= 2 GPUs: torch.distributed.run launches 2 ranks of the sharded step (dense and banded,
  1d and 2d, L = 512) and rank 0 compares C and S_A with the oracle (1e-10 / 1e-8) and with the
  single-GPU emulation of the same two shards (1e-12), click counts equal.  Skipped on one GPU
  (the pool grants one GPU per run; tests/test_comm_plan.py covers the schedule on CPU).
- On one GPU: the NCCL watchdog (csrc/watchdog.cu) turns a collective that never completes into
  TRAJ_ENCCL within its deadline instead of a hang (a one-rank communicator, the test hook
  TRAJ_WATCHDOG_TEST_STALL standing in for the missing peer)."""
import json
import os
import subprocess
import sys
import time

import pytest

from conftest import ROOT

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


def test_nccl_watchdog_aborts_a_stalled_collective(P, monkeypatch):
    monkeypatch.setenv("TRAJ_WATCHDOG_TEST_STALL", "1")
    monkeypatch.setenv("TRAJ_NCCL_TIMEOUT_S", "2")
    tr = P.Trajectories(256, 1, "homodyne", [1.0], seed=1, shard_size=1, shard_rank=0,
                        nccl_id=P.traj_nccl_unique_id())
    t0 = time.time()
    tr.step(1)                         # enqueues the never-completing "collective", returns
    assert time.time() - t0 < 1.0
    with pytest.raises(P.TrajError) as e:
        tr.failed(0)                   # waits on the stream: released by the watchdog's abort
    assert e.value.status == 5 and "watchdog" in str(e.value)
    assert time.time() - t0 < 30.0
    with pytest.raises(P.TrajError) as e:
        tr.step(1)                     # the communicator stays aborted: every call says so
    assert e.value.status == 5
    tr.close()


@pytest.mark.parametrize("L,Ly,protocol,gamma,propagator", [
    (512, 1, "projective", 2.0, "dense"),
    (512, 1, "homodyne", 1.0, "banded"),
    (576, 24, "projective", 3.0, "dense"),
    (576, 24, "homodyne", 1.5, "banded"),
])
def test_row_sharded_two_ranks_match_oracle_and_emulation(P, L, Ly, protocol, gamma, propagator):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (this pool grants one per run)")
    port = 29800 + os.getpid() % 100
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "mp_shard_worker.py"), str(L), str(Ly), protocol, str(gamma),
                        "6", propagator],
                       capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=dict(os.environ, TRAJ_NCCL_TIMEOUT_S="120"))
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["dC_oracle"] < 1e-10 and d["dS_oracle"] < 1e-8, d
    assert d["dC_emulation"] < 1e-12, d
    assert d["clicks"] == d["clicks_emulation"] == d["clicks_oracle"], d
