"""B200-native quantum-trajectory step for monitored free fermions (arXiv 2508.18468).

The product is ``libtraj.so`` (C-ABI, ``include/traj.h``).  This package is its thin
Python binding: ctypes marshalling plus torch for device memory and streams.  There
is no CPU fallback: loading fails loudly if the extension is missing.
"""
from .binding import (  # noqa: F401
    TRAJ_HOMODYNE,
    TRAJ_PROJECTIVE,
    TrajError,
    Trajectories,
    lib,
    load_library,
    traj_chol_inverse,
    traj_kernel_launches,
    traj_get_zgemm_algorithm,
    traj_nccl_unique_id,
    traj_comm_plan,
    traj_set_zgemm_algorithm,
    traj_zgemm,
    traj_dgemm,
)
