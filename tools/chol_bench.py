"""Time traj_chol_inverse at n = N of c3 (8192): eager vs replayed from a CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_18468_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
U = torch.randn(2 * n, n, dtype=torch.complex128, device="cuda")
G0 = torch.empty(n, n, dtype=torch.complex128, device="cuda")
P.traj_zgemm(1, 0, U, U, G0)
G = G0.clone()
X = torch.empty_like(G)
lib = P.lib()
scratch = torch.empty(int(lib.traj_chol_scratch_bytes(n, 1)) + 256, dtype=torch.uint8, device="cuda")
failed = torch.zeros(1, dtype=torch.int32, device="cuda")
sp = (scratch.data_ptr() + 255) // 256 * 256


def run(stream):
    G.copy_(G0)
    lib.traj_chol_inverse(stream, n, G.data_ptr(), n, n * n, X.data_ptr(), n, n * n, 1, sp, failed.data_ptr())


st = torch.cuda.current_stream().cuda_stream
run(st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
l0 = P.traj_kernel_launches()
e0.record()
for _ in range(3):
    run(st)
e1.record()
e1.synchronize()
launches = (P.traj_kernel_launches() - l0) / 3
eager = e0.elapsed_time(e1) / 3
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    run(s.cuda_stream)
g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(3):
    g.replay()
e1.record()
e1.synchronize()
graph = e0.elapsed_time(e1) / 3
# copy-only baseline
e0.record()
for _ in range(3):
    G.copy_(G0)
e1.record()
e1.synchronize()
cp = e0.elapsed_time(e1) / 3
fl = 8.0 / 3.0 * n ** 3
print(f"n={n} launches/call={launches:.0f} eager={eager - cp:.2f} ms graph={graph - cp:.2f} ms "
      f"({fl / (graph - cp) / 1e9:.1f} TF/s at graph) copy={cp:.2f} ms failed={failed.item()}")
Xr = X.cpu()
Gr = G0.cpu()
err = (Xr.conj().T @ Gr @ Xr - torch.eye(n, dtype=torch.complex128)).abs().max().item()
print("max|X^H G X - I| =", err)
