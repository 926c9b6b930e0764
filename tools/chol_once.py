import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2508_18468_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
U = torch.randn(2 * n, n, dtype=torch.complex128, device="cuda")
G0 = torch.empty(n, n, dtype=torch.complex128, device="cuda")
P.traj_zgemm(1, 0, U, U, G0)
G = G0.clone(); X = torch.empty_like(G)
lib = P.lib()
scratch = torch.empty(int(lib.traj_chol_scratch_bytes(n, 1)) + 256, dtype=torch.uint8, device="cuda")
failed = torch.zeros(1, dtype=torch.int32, device="cuda")
sp = (scratch.data_ptr() + 255) // 256 * 256
st = torch.cuda.current_stream().cuda_stream
for it in range(2):
    G.copy_(G0)
    if it == 1: torch.cuda.nvtx.range_push("chol")
    lib.traj_chol_inverse(st, n, G.data_ptr(), n, n * n, X.data_ptr(), n, n * n, 1, sp, failed.data_ptr())
    if it == 1: torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
