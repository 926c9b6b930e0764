"""Vendor reference for the FP64 denominators: cuBLAS ZGEMM/DGEMM via torch.matmul."""
import torch, os, subprocess
def bench(dtype, m, n, k, flop_per_mac):
    a = torch.randn(m, k, dtype=dtype, device="cuda"); b = torch.randn(k, n, dtype=dtype, device="cuda")
    for _ in range(2): torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(5):
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"{dtype} {m}x{n}x{k}: {flop_per_mac*m*n*k/best/1e9:.2f} TFLOP/s ({best:.2f} ms)")
bench(torch.float64, 8192, 8192, 8192, 2)
bench(torch.complex128, 8192, 8192, 8192, 8)
bench(torch.complex128, 16384, 8192, 16384, 8)
print("host cores:", len(os.sched_getaffinity(0)))
print(subprocess.run("lscpu | head -20", shell=True, capture_output=True, text=True).stdout)
import numpy as np
np.show_config()
