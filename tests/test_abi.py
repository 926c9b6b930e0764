"""The C-ABI library builds, loads and exports every symbol include/traj.h declares (CPU only:
no compute calls; without a GPU the device-needing calls must fail loudly, never fall back)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "traj.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(traj_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2508_18468_b200 import build
    build.build()
    from paper_2508_18468_b200 import binding
    return binding.load_library()


def test_header_declares_the_boundary():
    names = declared_functions()
    for core in ("traj_init", "traj_step", "traj_entropy", "traj_mutual_info", "traj_destroy",
                 "traj_workspace_bytes", "traj_zgemm", "traj_chol_inverse"):
        assert core in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    from paper_2508_18468_b200 import binding
    assert set(declared_functions()) == set(binding.EXPORTS)


def test_sass_is_sm100a_with_dmma_and_tma(lib):
    import subprocess
    from paper_2508_18468_b200.binding import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA.8x8x4" in out          # FP64 tensor pipe
    assert "UTMALDG" in out             # TMA loads


def test_strerror(lib):
    assert lib.traj_strerror(2) == b"invalid configuration"


def _cfg(**kw):
    from paper_2508_18468_b200.binding import TrajConfig
    g = np.array([0.5])
    c = TrajConfig(dim=1, Lx=64, Ly=1, N=32, J=1.0, dt=0.05, protocol=0, init=0, seed=0, n_traj=1, traj_base=0,
                   gamma=g.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), shard_rank=0, shard_size=1)
    for k, v in kw.items():
        setattr(c, k, v)
    return c, g


@pytest.mark.parametrize("field,value", [("N", 31), ("Lx", 63), ("dt", 0.0), ("protocol", 7), ("dim", 3),
                                         ("n_traj", 0), ("shard_size", 3), ("shard_rank", 1)])
def test_config_validation(lib, field, value):
    c, _keep = _cfg(**{field: value})
    if field == "Lx":
        c.N = 31
    out = ctypes.c_size_t(0)
    assert lib.traj_workspace_bytes(ctypes.byref(c), ctypes.byref(out)) == 2


def test_projective_rate_bound(lib):
    from paper_2508_18468_b200.binding import TrajConfig
    c, g = _cfg()
    g[0] = 30.0            # gamma*dt = 1.5 > 1
    out = ctypes.c_size_t(0)
    assert lib.traj_workspace_bytes(ctypes.byref(c), ctypes.byref(out)) == 2


def test_no_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c, _keep = _cfg()
    h = ctypes.c_void_p()
    assert lib.traj_init(ctypes.byref(c), ctypes.byref(h)) == 4      # TRAJ_ECUDA
    assert h.value is None


def test_sharding_needs_single_trajectory(lib):
    c, g = _cfg(shard_size=2)
    g2 = np.array([0.5, 0.5])
    c.gamma = g2.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    c.n_traj = 2
    out = ctypes.c_size_t(0)
    assert lib.traj_workspace_bytes(ctypes.byref(c), ctypes.byref(out)) == 2


def test_phase_names_match_the_header():
    """binding.PHASES sizes the buffers traj_phase_times fills: one name per TRAJ_PH_* entry."""
    txt = open(HEADER).read()
    n = int(re.search(r"TRAJ_NPHASES\s*=\s*(\d+)", txt).group(1))
    ids = [int(v) for v in re.findall(r"TRAJ_PH_[A-Z_0-9]+\s*=\s*(\d+)", txt)]
    from paper_2508_18468_b200 import binding
    assert len(binding.PHASES) == n == len(ids) and sorted(ids) == list(range(n))
