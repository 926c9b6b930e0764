"""One call of each modular product at the c3 shapes (for an ncu launch list)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2508_18468_b200 as P
P.load_library()
lib = P.lib()
L = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
N = L // 2
s = int(sys.argv[2]) if len(sys.argv) > 2 else 16
st = torch.cuda.current_stream().cuda_stream
K = torch.randn(L, L, dtype=torch.complex128, device="cuda")
U = torch.randn(L, N, dtype=torch.complex128, device="cuda")
X = torch.triu(torch.randn(N, N, dtype=torch.complex128, device="cuda"))
C = torch.empty(L, N, dtype=torch.complex128, device="cuda")
G = torch.empty(N, N, dtype=torch.complex128, device="cuda")
assert lib.traj_zgemm_ozaki(st, 0, L, N, L, K.data_ptr(), L, U.data_ptr(), N, C.data_ptr(), N, s, 0) == 0
assert lib.traj_zgemm_ozaki(st, 1, N, N, L, U.data_ptr(), N, U.data_ptr(), N, G.data_ptr(), N, s, 16) == 0
assert lib.traj_zgemm_ozaki(st, 0, L, N, N, U.data_ptr(), N, X.data_ptr(), N, C.data_ptr(), N, s, 4) == 0
torch.cuda.synchronize()
print("ok")
