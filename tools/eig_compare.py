"""Hermitian eigenvalues-only at the observables' sizes: cusolverDnZheevd (the library's call) vs
cusolverDnXsyevd (64-bit API) vs torch.linalg.eigvalsh.  Usage: python tools/eig_compare.py [n]"""
import ctypes, glob, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def _load(name):
    import nvidia
    for base in nvidia.__path__:
        hits = sorted(glob.glob(os.path.join(base, "*", "lib", name + "*")))
        if hits:
            return ctypes.CDLL(hits[0])
    return ctypes.CDLL(name)


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
torch.manual_seed(0)
Z = torch.randn(2 * n, n, dtype=torch.complex128, device="cuda")
H0 = (Z.conj().T @ Z) / (2 * n)
H = H0.clone()
cus = _load("libcusolver.so")
h = ctypes.c_void_p()
assert cus.cusolverDnCreate(ctypes.byref(h)) == 0
st = torch.cuda.current_stream().cuda_stream
assert cus.cusolverDnSetStream(h, ctypes.c_void_p(st)) == 0
w = torch.empty(n, dtype=torch.float64, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
lw = ctypes.c_int()
NOVEC, LOWER = 0, 0
assert cus.cusolverDnZheevd_bufferSize(h, NOVEC, LOWER, n, ctypes.c_void_p(H.data_ptr()), n,
                                       ctypes.c_void_p(w.data_ptr()), ctypes.byref(lw)) == 0
work = torch.empty(lw.value, dtype=torch.complex128, device="cuda")


def zheevd():
    H.copy_(H0)
    assert cus.cusolverDnZheevd(h, NOVEC, LOWER, n, ctypes.c_void_p(H.data_ptr()), n, ctypes.c_void_p(w.data_ptr()),
                                ctypes.c_void_p(work.data_ptr()), lw, ctypes.c_void_p(info.data_ptr())) == 0


params = ctypes.c_void_p()
assert cus.cusolverDnCreateParams(ctypes.byref(params)) == 0
C64F, R64F = 5, 1
dws, hws = ctypes.c_size_t(), ctypes.c_size_t()
assert cus.cusolverDnXsyevd_bufferSize(h, params, NOVEC, LOWER, ctypes.c_int64(n), C64F, ctypes.c_void_p(H.data_ptr()),
                                       ctypes.c_int64(n), R64F, ctypes.c_void_p(w.data_ptr()), C64F,
                                       ctypes.byref(dws), ctypes.byref(hws)) == 0
dwork = torch.empty(max(dws.value, 1), dtype=torch.uint8, device="cuda")
hwork = ctypes.create_string_buffer(max(hws.value, 1))


def xsyevd():
    H.copy_(H0)
    assert cus.cusolverDnXsyevd(h, params, NOVEC, LOWER, ctypes.c_int64(n), C64F, ctypes.c_void_p(H.data_ptr()),
                                ctypes.c_int64(n), R64F, ctypes.c_void_p(w.data_ptr()), C64F,
                                ctypes.c_void_p(dwork.data_ptr()), dws, hwork, hws,
                                ctypes.c_void_p(info.data_ptr())) == 0


copy = timed(lambda: H.copy_(H0))
res = {"n": n, "Zheevd_ms": timed(zheevd) - copy, "Xsyevd_ms": timed(xsyevd) - copy,
       "torch_eigvalsh_ms": timed(lambda: torch.linalg.eigvalsh(H0))}
print(res)
