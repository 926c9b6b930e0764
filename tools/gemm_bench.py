"""Time traj_zgemm variants at the c3 shapes with CUDA events (and compare cuBLAS ZGEMM)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_18468_b200 as P  # noqa: E402
from paper_2508_18468_b200 import binding as b  # noqa: E402

L, N = int(os.environ.get("GB_L", 16384)), int(os.environ.get("GB_N", 8192))
only = sys.argv[1:]
U = (torch.randn(L, N, dtype=torch.complex128, device="cuda"))
K = torch.randn(L, L, dtype=torch.complex128, device="cuda")
X = torch.triu(torch.randn(N, N, dtype=torch.complex128, device="cuda"))
G = torch.empty(N, N, dtype=torch.complex128, device="cuda")
O = torch.empty(L, N, dtype=torch.complex128, device="cuda")


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


cases = {
    "NN_KU": (lambda: P.traj_zgemm(0, 0, K, U, O), 8.0 * L * L * N),
    "CN_herk_upper": (lambda: P.traj_zgemm(1, 0, U, U, G, flags=b.TRAJ_C_UPPER), 4.0 * L * N * N),
    "CN_full": (lambda: P.traj_zgemm(1, 0, U, U, G), 8.0 * L * N * N),
    "NN_trmm": (lambda: P.traj_zgemm(0, 0, U, X, O, flags=b.TRAJ_TRI_B_UPPER), 4.0 * L * N * N),
    "NC_full": (lambda: P.traj_zgemm(0, 1, U[:N], U[:N], G), 8.0 * N * N * N),
    "cublas_KU": (lambda: torch.matmul(K, U, out=O), 8.0 * L * L * N),
    "cublas_herk_as_gemm": (lambda: torch.matmul(U.conj().T, U, out=G), 8.0 * L * N * N),
}
for name, (fn, fl) in cases.items():
    if only and name not in only:
        continue
    ms = t(fn)
    print(f"{name:22s} {ms:9.2f} ms  {fl / ms / 1e9:7.2f} TF/s")
