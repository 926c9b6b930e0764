"""ctypes binding of libtraj.so (include/traj.h): argument marshalling only.

Every step of the trajectory path runs in the library's CUDA kernels; torch only
allocates the workspace and provides the stream.  Names follow the C-ABI.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtraj.so")

TRAJ_PROJECTIVE = 0
TRAJ_HOMODYNE = 1
TRAJ_HOMODYNE_RK4 = 2
TRAJ_PROJECTIVE_EVENTS = 3
TRAJ_INIT_NEEL = 0
TRAJ_INIT_CHECKERBOARD = 1
TRAJ_PROP_DENSE, TRAJ_PROP_BANDED = 0, 1
TRAJ_TRI_A_UPPER, TRAJ_TRI_A_LOWER, TRAJ_TRI_B_UPPER, TRAJ_TRI_B_LOWER, TRAJ_C_UPPER = 1, 2, 4, 8, 16
PHASES = ("propagate", "monitor", "project", "gram", "chol", "trmm", "fused", "ku_mma", "gram_mma", "trmm_mma",
          "struct_factor")
# inside propagate / gram / trmm / chol: not additive
NESTED_PHASES = ("ku_mma", "gram_mma", "trmm_mma", "struct_factor")
STATUS = {0: "TRAJ_OK", 1: "TRAJ_EINVAL", 2: "TRAJ_ECONFIG", 3: "TRAJ_ENUMERIC", 4: "TRAJ_ECUDA",
          5: "TRAJ_ENCCL", 6: "TRAJ_EDOMAIN"}


class TrajConfig(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32),
        ("Lx", ctypes.c_int64),
        ("Ly", ctypes.c_int64),
        ("N", ctypes.c_int64),
        ("J", ctypes.c_double),
        ("dt", ctypes.c_double),
        ("protocol", ctypes.c_int32),
        ("init", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("n_traj", ctypes.c_int64),
        ("traj_base", ctypes.c_int64),
        ("gamma", ctypes.POINTER(ctypes.c_double)),
        ("shard_rank", ctypes.c_int32),
        ("shard_size", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p),
        ("stream", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_size_t),
        ("propagator", ctypes.c_int32),
        ("orthonormalizer", ctypes.c_int32),
    ]


class TrajError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_SIGS = {
    "traj_workspace_bytes": (ctypes.c_int, [ctypes.POINTER(TrajConfig), ctypes.POINTER(ctypes.c_size_t)]),
    "traj_init": (ctypes.c_int, [ctypes.POINTER(TrajConfig), ctypes.POINTER(_P)]),
    "traj_step": (ctypes.c_int, [_P, _I64]),
    "traj_orthonormalize": (ctypes.c_int, [_P]),
    "traj_entropy": (ctypes.c_int, [_P, ctypes.POINTER(_I64), _I64, ctypes.POINTER(_D)]),
    "traj_mutual_info": (ctypes.c_int, [_P, ctypes.POINTER(_I64), _I64, ctypes.POINTER(_I64), _I64,
                                        ctypes.POINTER(_D)]),
    "traj_density_correlation": (ctypes.c_int, [_P, _I64, ctypes.POINTER(_D)]),
    "traj_particle_covariance": (ctypes.c_int, [_P, ctypes.POINTER(_I64), _I64, ctypes.POINTER(_I64), _I64,
                                                ctypes.POINTER(_D)]),
    "traj_occupations": (ctypes.c_int, [_P, _P]),
    "traj_correlation_rows": (ctypes.c_int, [_P, _I64, _I64, _I64, _P]),
    "traj_get_state": (ctypes.c_int, [_P, _I64, _P]),
    "traj_set_state": (ctypes.c_int, [_P, _I64, _P]),
    "traj_get_step": (ctypes.c_int, [_P, ctypes.POINTER(_I64)]),
    "traj_set_step": (ctypes.c_int, [_P, _I64]),
    "traj_failed": (ctypes.c_int, [_P, _I64, ctypes.POINTER(ctypes.c_int32)]),
    "traj_last_clicks": (ctypes.c_int, [_P, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "traj_cqr2_fallbacks": (ctypes.c_int, [_P, ctypes.POINTER(_I64)]),
    "traj_gram_deviation": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_double)]),
    "traj_probe_orthonormality": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_double)]),
    "traj_lowrank_stats": (ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                                          ctypes.POINTER(_I64)]),
    "traj_profile": (ctypes.c_int, [_P, ctypes.c_int]),
    "traj_phase_times": (ctypes.c_int, [_P, ctypes.POINTER(_D), ctypes.POINTER(_I64)]),
    "traj_ozaki_info": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int32)]),
    "traj_kernel_launches": (ctypes.c_longlong, []),
    "traj_destroy": (ctypes.c_int, [_P]),
    "traj_last_error": (ctypes.c_char_p, [_P]),
    "traj_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "traj_zgemm": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _I64, _I64, _I64, _D, _D, _P, _I64, _I64, _P, _I64,
                                  _I64, _D, _P, _I64, _I64, _I64, ctypes.c_int]),
    "traj_dgemm": (ctypes.c_int, [_P, _I64, _I64, _I64, _D, _P, _I64, _I64, _P, _I64, _I64, _D, _P, _I64, _I64, _I64]),
    "traj_igemm": (ctypes.c_int, [_P, _I64, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _I64, _P,
                                  ctypes.c_int, ctypes.c_int]),
    "traj_zgemm_ozaki": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, ctypes.c_int,
                                        ctypes.c_int]),
    "traj_ozaki_constants": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                            ctypes.POINTER(_D), ctypes.POINTER(_D), ctypes.POINTER(_D)]),
    "traj_ozaki_roots": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int32)]),
    "traj_shard_info": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                       ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "traj_nccl_unique_id": (ctypes.c_int, [_P]),
    "traj_comm_plan": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _I64, ctypes.POINTER(_I64), _I64]),
    "traj_set_zgemm_algorithm": (ctypes.c_int, [ctypes.c_int]),
    "traj_get_zgemm_algorithm": (ctypes.c_int, []),
    "traj_chol_scratch_bytes": (ctypes.c_size_t, [_I64, _I64]),
    "traj_chol_inverse": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _P, _I64, _I64, _I64, _P, _P]),
}
EXPORTS = tuple(_SIGS)


def load_library(path: str = LIB_PATH):
    """Load libtraj.so; raises (never falls back) if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        lib_ = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib_, name)
            f.restype = res
            f.argtypes = args
        _lib = lib_
    return _lib


def lib():
    return load_library()


def _check(status: int, handle=None):
    if status != 0:
        msg = lib().traj_last_error(handle)
        raise TrajError(status, msg.decode() if msg else "")


def traj_kernel_launches() -> int:
    return int(lib().traj_kernel_launches())


def _ptr(t) -> int:
    return int(t.data_ptr())


def traj_set_zgemm_algorithm(algo: str | int):
    """"3m" (1, the default: Gauss, three real DMMA products) or "4m" (0) complex multiplication in
    every contraction (process-wide; the environment TRAJ_ZGEMM_3M=0 sets 4m at load)."""
    a = {"4m": 0, "3m": 1}.get(algo, algo) if isinstance(algo, str) else int(algo)
    _check(lib().traj_set_zgemm_algorithm(a))


def traj_get_zgemm_algorithm() -> str:
    return "3m" if lib().traj_get_zgemm_algorithm() == 1 else "4m"


def traj_nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 creates it; the caller broadcasts it)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().traj_nccl_unique_id(buf))
    return buf.raw


def traj_comm_plan(kind: int, P: int, rank: int, n: int = 0) -> np.ndarray:
    """The row-sharded step's communication schedule for one rank (host data, no GPU): kind 0 the
    ring exchange of the propagate, 1 the halo exchange, 2 the distributed Cholesky's broadcasts.
    Rows (group, op, peer, slot, block) for kinds 0/1, (root, rows, cols) for kind 2."""
    w = 3 if kind == 2 else 5
    cnt = lib().traj_comm_plan(kind, P, rank, n, None, 0)
    if cnt < 0:
        _check(-cnt)
    out = np.zeros(max(cnt, 1) * w, dtype=np.int64)
    lib().traj_comm_plan(kind, P, rank, n, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), cnt)
    return out[:cnt * w].reshape(cnt, w)


def traj_zgemm(opA, opB, A, B, C, *, alpha=1.0, beta=0.0, flags=0, M=None, N=None, K=None, stream=None):
    """C = alpha op(A) op(B) + beta C on torch complex128 CUDA tensors (2d, or 3d = batch)."""
    import torch
    lib_ = lib()
    batched = C.dim() == 3
    Ab = A if A.dim() == 3 else A.unsqueeze(0)
    Bb = B if B.dim() == 3 else B.unsqueeze(0)
    Cb = C if batched else C.unsqueeze(0)
    batch = Cb.shape[0]
    M = Cb.shape[1] if M is None else M
    N = Cb.shape[2] if N is None else N
    K = (Ab.shape[2] if opA == 0 else Ab.shape[1]) if K is None else K
    for t in (Ab, Bb, Cb):
        assert t.dtype == torch.complex128 and t.is_cuda and t.stride(-1) == 1
    sA = Ab.stride(0) if Ab.shape[0] > 1 else 0
    sB = Bb.stride(0) if Bb.shape[0] > 1 else 0
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    a = complex(alpha)
    _check(lib_.traj_zgemm(st, opA, opB, M, N, K, a.real, a.imag, _ptr(Ab), Ab.stride(-2), sA, _ptr(Bb),
                           Bb.stride(-2), sB, float(beta), _ptr(Cb), Cb.stride(-2), Cb.stride(0), batch, flags))
    return C


def traj_dgemm(A, B, C, *, alpha=1.0, beta=0.0, stream=None):
    """C = alpha A B + beta C on torch float64 CUDA tensors (2d, or 3d = batch), row-major, no transposes."""
    import torch
    lib_ = lib()
    Ab = A if A.dim() == 3 else A.unsqueeze(0)
    Bb = B if B.dim() == 3 else B.unsqueeze(0)
    Cb = C if C.dim() == 3 else C.unsqueeze(0)
    for t in (Ab, Bb, Cb):
        assert t.dtype == torch.float64 and t.is_cuda and t.stride(-1) == 1
    batch, M, N = Cb.shape
    K = Ab.shape[2]
    sA = Ab.stride(0) if Ab.shape[0] > 1 else 0
    sB = Bb.stride(0) if Bb.shape[0] > 1 else 0
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _check(lib_.traj_dgemm(st, M, N, K, float(alpha), _ptr(Ab), Ab.stride(-2), sA, _ptr(Bb), Bb.stride(-2), sB,
                           float(beta), _ptr(Cb), Cb.stride(-2), Cb.stride(0), batch))
    return C


def traj_chol_inverse(G, X, failed=None, stream=None):
    """X_b = R^-1 with G_b = R^dag R (upper triangle of G read; its lower triangle is clobbered)."""
    import torch
    lib_ = lib()
    Gb = G if G.dim() == 3 else G.unsqueeze(0)
    Xb = X if X.dim() == 3 else X.unsqueeze(0)
    batch, n = Gb.shape[0], Gb.shape[1]
    scratch = torch.empty(int(lib_.traj_chol_scratch_bytes(n, batch)) + 256, dtype=torch.uint8, device=G.device)
    if failed is None:
        failed = torch.zeros(batch, dtype=torch.int32, device=G.device)
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    sp = (_ptr(scratch) + 255) // 256 * 256
    _check(lib_.traj_chol_inverse(st, n, _ptr(Gb), Gb.stride(-2), Gb.stride(0), _ptr(Xb), Xb.stride(-2),
                                  Xb.stride(0), batch, sp, _ptr(failed)))
    return X, failed


class Trajectories:
    """A batch of trajectories on one GPU: the handle of ``traj_init``.

    Lx, Ly: lattice extents (Ly = 1 for the 1d ring); protocol: "projective" or
    "homodyne"; gammas: per-trajectory per-site rate; seed / traj_base: Philox key and
    global id of the first trajectory (reading Q9)."""

    def __init__(self, Lx: int, Ly: int = 1, protocol: str = "projective", gammas=(0.5,), dt: float = 0.05,
                 J: float = 1.0, seed: int = 0, traj_base: int = 0, device=None, stream=None,
                 shard_size: int = 1, shard_rank: int = 0, nccl_id: bytes | None = None,
                 propagator: str = "dense", orthonormalizer: str = "cqr2"):
        import torch
        self._torch = torch
        lib_ = lib()
        self.device = torch.device(device if device is not None else "cuda")
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.Lx, self.Ly = int(Lx), int(Ly)
        self.L = self.Lx * self.Ly
        self.N = self.L // 2
        self.gammas = np.ascontiguousarray(np.asarray(gammas, dtype=np.float64).ravel())
        self.n_traj = int(self.gammas.size)
        self.protocol = protocol
        cfg = TrajConfig()
        cfg.dim = 1 if self.Ly == 1 else 2
        cfg.Lx, cfg.Ly, cfg.N = self.Lx, self.Ly, self.N
        cfg.J, cfg.dt = float(J), float(dt)
        cfg.protocol = {"projective": TRAJ_PROJECTIVE, "homodyne": TRAJ_HOMODYNE,
                        "homodyne_rk4": TRAJ_HOMODYNE_RK4, "projective_events": TRAJ_PROJECTIVE_EVENTS}[protocol]
        cfg.init = TRAJ_INIT_NEEL if self.Ly == 1 else TRAJ_INIT_CHECKERBOARD
        cfg.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        cfg.n_traj = self.n_traj
        cfg.traj_base = int(traj_base)
        cfg.gamma = self.gammas.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        cfg.shard_rank, cfg.shard_size = int(shard_rank), int(shard_size)
        self._nccl_id = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        cfg.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p) if nccl_id is not None else None
        cfg.stream = self.stream.cuda_stream
        cfg.propagator = {"dense": TRAJ_PROP_DENSE, "banded": TRAJ_PROP_BANDED}[propagator]
        cfg.orthonormalizer = {"cqr2": 0, "lowrank": 1}[orthonormalizer]
        nbytes = ctypes.c_size_t(0)
        _check(lib_.traj_workspace_bytes(ctypes.byref(cfg), ctypes.byref(nbytes)))
        self.workspace = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=self.device)
        cfg.workspace = (_ptr(self.workspace) + 255) // 256 * 256
        cfg.workspace_bytes = nbytes.value
        self._cfg = cfg
        h = ctypes.c_void_p()
        _check(lib_.traj_init(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        P, nloc, r0, rows = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib_.traj_shard_info(h, ctypes.byref(P), ctypes.byref(nloc), ctypes.byref(r0), ctypes.byref(rows)))
        self.shard_size, self.local_shards, self.row0, self.rows = P.value, nloc.value, r0.value, rows.value

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib().traj_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _c(self, status):
        _check(status, self._h)

    # -- the step
    def step(self, n: int = 1):
        self._c(lib().traj_step(self._h, int(n)))

    def orthonormalize(self):
        self._c(lib().traj_orthonormalize(self._h))

    # -- observables
    @staticmethod
    def _sites(A):
        a = np.ascontiguousarray(np.asarray(A, dtype=np.int64).ravel())
        return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))

    def entropy(self, A) -> np.ndarray:
        a, pa = self._sites(A)
        out = np.zeros(self.n_traj)
        self._c(lib().traj_entropy(self._h, pa, a.size, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def mutual_info(self, A, B) -> np.ndarray:
        a, pa = self._sites(A)
        b, pb = self._sites(B)
        out = np.zeros(self.n_traj)
        self._c(lib().traj_mutual_info(self._h, pa, a.size, pb, b.size,
                                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def density_correlation(self, traj: int = 0) -> np.ndarray:
        """C(r), Eq. (2), r = 0..L-1 (entry 0 is NaN); 1d only."""
        out = np.zeros(self.L)
        self._c(lib().traj_density_correlation(self._h, traj, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def particle_covariance(self, A, B) -> np.ndarray:
        """G_AB, Eq. (5), for every trajectory."""
        a, pa = self._sites(A)
        b, pb = self._sites(B)
        out = np.zeros(self.n_traj)
        self._c(lib().traj_particle_covariance(self._h, pa, a.size, pb, b.size,
                                               out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def occupations(self):
        """n_i of the rows this handle holds: [n_traj][rows] (rows = L unless row-sharded)."""
        n = self._torch.empty((self.n_traj, self.rows), dtype=self._torch.float64, device=self.device)
        self._c(lib().traj_occupations(self._h, _ptr(n)))
        return n

    def correlation_rows(self, traj: int, row0: int, nrows: int):
        C = self._torch.empty((nrows, self.L), dtype=self._torch.complex128, device=self.device)
        self._c(lib().traj_correlation_rows(self._h, traj, row0, nrows, _ptr(C)))
        return C

    def correlation(self, traj: int = 0):
        return self.correlation_rows(traj, 0, self.L)

    def get_state(self, traj: int = 0, out=None):
        if out is None:
            out = self._torch.empty((self.rows, self.N), dtype=self._torch.complex128, device=self.device)
        self._c(lib().traj_get_state(self._h, traj, _ptr(out)))
        return out

    def set_state(self, traj: int, U):
        U = U.contiguous()
        assert U.dtype == self._torch.complex128 and tuple(U.shape) == (self.rows, self.N)
        self._c(lib().traj_set_state(self._h, traj, _ptr(U)))

    def failed(self, traj: int) -> bool:
        f = ctypes.c_int32(0)
        self._c(lib().traj_failed(self._h, traj, ctypes.byref(f)))
        return bool(f.value)

    def last_clicks(self, traj: int = 0):
        a, b = ctypes.c_int64(0), ctypes.c_int64(0)
        self._c(lib().traj_last_clicks(self._h, traj, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    @property
    def step_index(self) -> int:
        s = ctypes.c_int64(0)
        self._c(lib().traj_get_step(self._h, ctypes.byref(s)))
        return s.value

    @step_index.setter
    def step_index(self, v: int):
        self._c(lib().traj_set_step(self._h, int(v)))

    def cqr2_fallbacks(self) -> int:
        n = ctypes.c_int64(0)
        self._c(lib().traj_cqr2_fallbacks(self._h, ctypes.byref(n)))
        return n.value

    def gram_deviation(self):
        """max|G2 - I| measured by the most recent CholeskyQR2 second pass, per trajectory."""
        import numpy as np
        out = np.zeros(self.n_traj, dtype=np.float64)
        self._c(lib().traj_gram_deviation(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def probe_orthonormality(self):
        """Estimated ||U_t^dag U_t - I||_F per trajectory (4 random unit-modulus probes)."""
        import numpy as np
        out = np.zeros(self.n_traj, dtype=np.float64)
        self._c(lib().traj_probe_orthonormality(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def lowrank_stats(self) -> dict:
        """Counters of the low-rank orthonormaliser: Newton-Schulz iterations, fallbacks to
        CholeskyQR2, orthonormality probes and the refinements they triggered."""
        v = [ctypes.c_int64(0) for _ in range(4)]
        self._c(lib().traj_lowrank_stats(self._h, *[ctypes.byref(x) for x in v]))
        return dict(zip(("newton_iters", "fallbacks", "probes", "refinements"), (x.value for x in v)))

    # -- profiling
    def profile(self, enable: bool = True):
        self._c(lib().traj_profile(self._h, 1 if enable else 0))

    def ozaki_info(self):
        """(K U on the INT8 modular path, Gram/TRMM on it, modulus count)."""
        out = (ctypes.c_int32 * 3)()
        self._c(lib().traj_ozaki_info(self._h, out))
        return bool(out[0]), bool(out[1]), int(out[2])

    def phase_times(self):
        ms = (ctypes.c_double * len(PHASES))()
        ln = (ctypes.c_int64 * len(PHASES))()
        self._c(lib().traj_phase_times(self._h, ms, ln))
        return {p: (ms[i], ln[i]) for i, p in enumerate(PHASES)}
