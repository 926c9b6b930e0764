"""Same-shape library denominators for the c3 step's contractions (SURVEY §8(d) "against ...
(iii) cuBLAS ZGEMM on the same shape").

Times, with CUDA events on one stream after warm-up:
  K U        (L x L) (L x N), row-major      : traj_zgemm (interleaved 3M) and traj_dgemm x3 (planar 3M,
                                               the propagator's path) vs cublasZgemm / cublasZgemm3m /
                                               cuBLAS Dgemm on the same three real products
  U^dag U    (N x L) (L x N) (full, no tri)  : traj_zgemm  vs cublasZgemm / cublasZgemm3m
  G = R^dag R, X = R^-1 (n = N)              : traj_chol_inverse vs cusolverDnZpotrf + cusolverDnXtrtri
cuBLAS / cuSOLVER are column-major: a row-major C = A B is the column-major C^T = B^T A^T.
Prints one JSON object.  Usage: python tools/library_compare.py [L] [reps]
"""
import ctypes
import glob
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_18468_b200 as P  # noqa: E402


def _load(name):
    import nvidia
    for base in nvidia.__path__:
        hits = sorted(glob.glob(os.path.join(base, "*", "lib", name + "*")))
        if hits:
            return ctypes.CDLL(hits[0])
    return ctypes.CDLL(name)


class Z(ctypes.Structure):
    _fields_ = [("x", ctypes.c_double), ("y", ctypes.c_double)]


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    N = L // 2
    dev = "cuda"
    st = torch.cuda.current_stream().cuda_stream
    cublas = _load("libcublas.so")
    h = ctypes.c_void_p()
    assert cublas.cublasCreate_v2(ctypes.byref(h)) == 0
    assert cublas.cublasSetStream_v2(h, ctypes.c_void_p(st)) == 0
    one, zero = Z(1.0, 0.0), Z(0.0, 0.0)
    CUBLAS_OP_N, CUBLAS_OP_C = 0, 2
    torch.manual_seed(0)
    K = torch.randn(L, L, dtype=torch.complex128, device=dev)
    U = torch.randn(L, N, dtype=torch.complex128, device=dev)
    V = torch.empty(L, N, dtype=torch.complex128, device=dev)
    G = torch.empty(N, N, dtype=torch.complex128, device=dev)
    out = {"L": L, "N": N, "reps": reps, "device": torch.cuda.get_device_name()}

    def cub(fn, opa, opb, m, n, k, A, lda, B, ldb, C, ldc):
        p = ctypes.c_void_p
        r = fn(h, opa, opb, m, n, k, ctypes.byref(one), p(A.data_ptr()), lda, p(B.data_ptr()), ldb,
               ctypes.byref(zero), p(C.data_ptr()), ldc)
        assert r == 0, r

    # K U: column-major V^T (N x L) = U^T (N x L) K^T (L x L)
    f_ku = 8.0 * L * L * N
    ku = {
        "ours_interleaved_zgemm3m": lambda: P.traj_zgemm(0, 0, K, U, V),
        "cublasZgemm": lambda: cub(cublas.cublasZgemm_v2, CUBLAS_OP_N, CUBLAS_OP_N, N, L, L, U, N, K, L, V, N),
        "cublasZgemm3m": lambda: cub(cublas.cublasZgemm3m, CUBLAS_OP_N, CUBLAS_OP_N, N, L, L, U, N, K, L, V, N),
    }
    res = {}
    ref = None
    for name, fn in ku.items():
        ms = timed(fn, reps)
        torch.cuda.synchronize()
        if ref is None:
            ref = V.clone()
        err = (V - ref).abs().max().item() / ref.abs().max().item()
        res[name] = {"ms": ms, "tflops_8mnk": f_ku / ms / 1e9, "rel_diff_vs_ours": err}
    # planar 3M: the three real products (Kr Ur, Ki Ui, (Kr+Ki)(Ur+Ui)) as one batch-3 traj_dgemm,
    # the path the library's propagator takes; split/combine (2 x 0.8 ms at c3) timed with ours
    Kp = torch.stack([K.real, K.imag, K.real + K.imag]).contiguous()
    ldp = (N + 15) // 16 * 16
    Up = torch.zeros(3, L, ldp, dtype=torch.float64, device=dev)
    Up[0, :, :N], Up[1, :, :N], Up[2, :, :N] = U.real, U.imag, U.real + U.imag
    Pp = torch.empty(3, L, ldp, dtype=torch.float64, device=dev)

    def planar():
        r = lib.traj_dgemm(st, L, N, L, 1.0, Kp.data_ptr(), L, L * L, Up.data_ptr(), ldp, L * ldp, 0.0,
                           Pp.data_ptr(), ldp, L * ldp, 3)
        assert r == 0, r

    lib = P.lib()
    ms = timed(planar, reps)
    Vp = torch.complex(Pp[0, :, :N] - Pp[1, :, :N], Pp[2, :, :N] - Pp[0, :, :N] - Pp[1, :, :N])
    err = (Vp - ref).abs().max().item() / ref.abs().max().item()
    res["ours_planar_3x_dgemm"] = {"ms": ms, "tflops_8mnk": f_ku / ms / 1e9, "rel_diff_vs_ours": err,
                                   "note": "three real 16384x8192x16384 products in one batch-3 launch; the "
                                           "propagator adds a split and a combine pass (about 1.5 ms at c3)"}
    Kr, Ur = Kp, Up[:, :, :N].contiguous()
    Pr = torch.empty(3, L, N, dtype=torch.float64, device=dev)
    ms = timed(lambda: torch.bmm(Kr, Ur, out=Pr), reps)
    res["cublasDgemm_3_real_products"] = {"ms": ms, "tflops_8mnk": f_ku / ms / 1e9}
    del Kp, Up, Pp, Vp, Kr, Ur, Pr
    out["K_U"] = res
    del ref
    # U^dag U (full N x N): column-major G^T (N x N) = U^T (N x L) conj(U) (L x N)
    # row-major G = U^H U  <->  column-major G^T = U^T conj(U); with Ucm = U^T (N x L, ld N):
    # G^T = Ucm (Ucm)^H ... conjugated; compare |G| entries only (timing is what matters here).
    f_g = 8.0 * N * N * L
    gram = {
        "ours": lambda: P.traj_zgemm(1, 0, U, U, G),
        "cublasZgemm": lambda: cub(cublas.cublasZgemm_v2, CUBLAS_OP_N, CUBLAS_OP_C, N, N, L, U, N, U, N, G, N),
        "cublasZgemm3m": lambda: cub(cublas.cublasZgemm3m, CUBLAS_OP_N, CUBLAS_OP_C, N, N, L, U, N, U, N, G, N),
    }
    res = {}
    for name, fn in gram.items():
        ms = timed(fn, reps)
        res[name] = {"ms": ms, "tflops_8mnk": f_g / ms / 1e9}
    out["Udag_U_full"] = res
    del K, V
    torch.cuda.empty_cache()

    # Cholesky + triangular inverse of an SPD Gram (n = N)
    W = torch.randn(2 * N, N, dtype=torch.complex128, device=dev)
    G0 = torch.empty(N, N, dtype=torch.complex128, device=dev)
    P.traj_zgemm(1, 0, W, W, G0)
    del W
    Gw = G0.clone()
    X = torch.empty_like(G0)
    res = {}

    def ours():
        Gw.copy_(G0)
        P.traj_chol_inverse(Gw, X)

    copy_ms = timed(lambda: Gw.copy_(G0), reps)
    res["ours"] = {"ms": timed(ours, reps) - copy_ms}
    cus = _load("libcusolver.so")
    hs = ctypes.c_void_p()
    assert cus.cusolverDnCreate(ctypes.byref(hs)) == 0
    assert cus.cusolverDnSetStream(hs, ctypes.c_void_p(st)) == 0
    lwork = ctypes.c_int()
    UPPER_cm = 0  # CUBLAS_FILL_MODE_LOWER in column-major == upper triangle of the row-major G^T...
    # row-major G (Hermitian) read as column-major is G^T = conj(G); its lower triangle holds the
    # row-major upper triangle.  conj(G) = conj(R)^H conj(R) is factorised as L L^H with L lower.
    assert cus.cusolverDnZpotrf_bufferSize(hs, UPPER_cm, N, ctypes.c_void_p(Gw.data_ptr()), N,
                                           ctypes.byref(lwork)) == 0
    work = torch.empty(max(lwork.value, 1), dtype=torch.complex128, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    CUDA_C_64F = 5
    dws, hws = ctypes.c_size_t(), ctypes.c_size_t()
    assert cus.cusolverDnXtrtri_bufferSize(hs, UPPER_cm, 0, ctypes.c_int64(N), CUDA_C_64F,
                                           ctypes.c_void_p(Gw.data_ptr()), ctypes.c_int64(N), ctypes.byref(dws),
                                           ctypes.byref(hws)) == 0
    dwork = torch.empty(max(dws.value, 1), dtype=torch.uint8, device=dev)
    hwork = ctypes.create_string_buffer(max(hws.value, 1))

    def potrf():
        Gw.copy_(G0)
        r = cus.cusolverDnZpotrf(hs, UPPER_cm, N, ctypes.c_void_p(Gw.data_ptr()), N, ctypes.c_void_p(work.data_ptr()),
                                 lwork.value, ctypes.c_void_p(info.data_ptr()))
        assert r == 0, r

    def potrf_trtri():
        potrf()
        r = cus.cusolverDnXtrtri(hs, UPPER_cm, 0, ctypes.c_int64(N), CUDA_C_64F, ctypes.c_void_p(Gw.data_ptr()),
                                 ctypes.c_int64(N), ctypes.c_void_p(dwork.data_ptr()), dws, hwork, hws,
                                 ctypes.c_void_p(info.data_ptr()))
        assert r == 0, r

    res["cusolverDnZpotrf"] = {"ms": timed(potrf, reps) - copy_ms}
    res["cusolverDnZpotrf+Xtrtri"] = {"ms": timed(potrf_trtri, reps) - copy_ms}
    res["info"] = int(info.item())
    out["chol_inverse"] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()
