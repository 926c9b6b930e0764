"""Time the exact modular complex products (traj_zgemm_ozaki, scratch allocation and splits included)
against the DMMA complex GEMM (traj_zgemm, 3M) at the c3 shapes: K U, the Gram U^dag U (upper), and
U X with X upper triangular.  Also the max deviation between the two results."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2508_18468_b200 as P

P.load_library()
lib = P.lib()
L = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
N = L // 2
s = int(sys.argv[2]) if len(sys.argv) > 2 else 16
st = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda").manual_seed(0)


def rnd(m, n):
    return torch.complex(torch.randn(m, n, device="cuda", dtype=torch.float64, generator=g),
                         torch.randn(m, n, device="cuda", dtype=torch.float64, generator=g)) / (m ** 0.5)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


K = rnd(L, L)
U = rnd(L, N)
X = torch.triu(rnd(N, N))
C1 = torch.empty(L, N, dtype=torch.complex128, device="cuda")
C2 = torch.empty(L, N, dtype=torch.complex128, device="cuda")
G1 = torch.zeros(N, N, dtype=torch.complex128, device="cuda")
G2 = torch.zeros(N, N, dtype=torch.complex128, device="cuda")


def oz_ku():
    assert lib.traj_zgemm_ozaki(st, 0, L, N, L, K.data_ptr(), L, U.data_ptr(), N, C1.data_ptr(), N, s, 0) == 0


def dm_ku():
    assert lib.traj_zgemm(st, 0, 0, L, N, L, 1.0, 0.0, K.data_ptr(), L, 0, U.data_ptr(), N, 0, 0.0, C2.data_ptr(), N, 0, 1, 0) == 0


def oz_gram():
    assert lib.traj_zgemm_ozaki(st, 1, N, N, L, U.data_ptr(), N, U.data_ptr(), N, G1.data_ptr(), N, s, 16) == 0


def dm_gram():
    assert lib.traj_zgemm(st, 1, 0, N, N, L, 1.0, 0.0, U.data_ptr(), N, 0, U.data_ptr(), N, 0, 0.0, G2.data_ptr(), N, 0, 1, 16) == 0


def oz_trmm():
    assert lib.traj_zgemm_ozaki(st, 0, L, N, N, U.data_ptr(), N, X.data_ptr(), N, C1.data_ptr(), N, s, 4) == 0


def dm_trmm():
    assert lib.traj_zgemm(st, 0, 0, L, N, N, 1.0, 0.0, U.data_ptr(), N, 0, X.data_ptr(), N, 0, 0.0, C2.data_ptr(), N, 0, 1, 4) == 0


for name, a, b, fl in [("K U", oz_ku, dm_ku, 8.0 * L * L * N), ("Gram", oz_gram, dm_gram, 4.0 * L * N * N),
                       ("U X", oz_trmm, dm_trmm, 4.0 * L * N * N)]:
    ta = timeit(a)
    tb = timeit(b)
    if name == "Gram":
        d = (torch.triu(G1) - torch.triu(G2)).abs().max().item()
        ref = torch.triu(G2).abs().max().item()
    else:
        d = (C1 - C2).abs().max().item()
        ref = C2.abs().max().item()
    print(f"{name:5s} L={L} N={N} s={s}: ozaki {ta:8.2f} ms ({fl / ta / 1e9:6.1f} TF/s 8mnk-equiv)   dmma {tb:8.2f} ms"
          f"   max|diff| {d:.3e} (max|C| {ref:.3e})", flush=True)
