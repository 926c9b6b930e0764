"""Real FP64 DMMA GEMM (traj_dgemm): correctness against torch (cuBLAS DGEMM) and TF/s at the planar
3M shapes of c3's K.U (three real 16384 x 8192 x 16384 products as one batch of 3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2508_18468_b200 as P  # noqa: E402


def timed(fn, reps=3):
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


torch.manual_seed(0)
for (M, N, K) in [(300, 200, 100), (1000, 520, 777), (129, 17, 33)]:
    ldb = (N + 15) // 16 * 16
    A = torch.randn(M, K, dtype=torch.float64, device="cuda")
    Bf = torch.randn(K, ldb, dtype=torch.float64, device="cuda")
    B = Bf[:, :N]
    C = torch.randn(M, N + (N & 1), dtype=torch.float64, device="cuda")[:, :N] if False else torch.randn(M, N, dtype=torch.float64, device="cuda")
    C0 = C.clone()
    ref = 0.5 * (A @ B) + 2.0 * C0
    if N % 2:
        Cp = torch.zeros(M, N + 1, dtype=torch.float64, device="cuda")
        Cp[:, :N] = C0
        P.traj_dgemm(A, Bf[:, :N], Cp[:, :N], alpha=0.5, beta=2.0) if False else None
    lib = P.lib()
    st = torch.cuda.current_stream().cuda_stream
    ldc = N + (N & 1)
    Cbuf = torch.zeros(M, ldc, dtype=torch.float64, device="cuda")
    Cbuf[:, :N] = C0
    r = lib.traj_dgemm(st, M, N, K, 0.5, A.data_ptr(), K + (K & 1) if False else A.stride(0), 0, Bf.data_ptr(), ldb, 0,
                       2.0, Cbuf.data_ptr(), ldc, 0, 1)
    torch.cuda.synchronize()
    err = (Cbuf[:, :N] - ref).abs().max().item() / ref.abs().max().item() if r == 0 else None
    print(f"M={M} N={N} K={K} status={r} rel err={err}")
L, N = int(os.environ.get("GB_L", 16384)), int(os.environ.get("GB_N", 8192))
A = torch.randn(3, L, L, dtype=torch.float64, device="cuda")
B = torch.randn(3, L, N, dtype=torch.float64, device="cuda")
C = torch.empty(3, L, N, dtype=torch.float64, device="cuda")
ms = timed(lambda: P.traj_dgemm(A, B, C))
fl = 3 * 2.0 * L * L * N
print(f"batched 3 x {L}x{N}x{L}: {ms:.2f} ms  {fl / ms / 1e9:.2f} TF/s (pipe; 37.1 peak -> {fl / ms / 1e9 / 37.1:.3f}); "
      f"as planar 3M K.U: {8.0 * L * L * N / ms / 1e9:.2f} TF/s algorithmic")
ref = torch.bmm(A[:, :512], B)
print("rel err vs cuBLAS (first 512 rows):", ((C[:, :512] - ref).abs().max() / ref.abs().max()).item())
ms2 = timed(lambda: torch.bmm(A, B, out=C))
print(f"cuBLAS DGEMM batched: {ms2:.2f} ms  {fl / ms2 / 1e9:.2f} TF/s")
