"""Host-side transfer probes for the e2e path (diagnostic): D2H into registered (pinned)
pageable memory, int64 vs int32, and the THP setting."""
import ctypes, os, time
import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so")
print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
N = 207_513_882
dev64 = torch.empty(N, dtype=torch.int64, device="cuda")
dev32 = torch.empty(N, dtype=torch.int32, device="cuda")
host = np.ones(N, dtype=np.int64)  # faulted in
t0 = time.perf_counter()
rc = cudart.cudaHostRegister(ctypes.c_void_p(host.ctypes.data), ctypes.c_size_t(host.nbytes), 0)
print("register rc", rc, f"{(time.perf_counter()-t0)*1e3:.1f} ms")
cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cudart.cudaMemcpy(ctypes.c_void_p(host.ctypes.data), ctypes.c_void_p(dev64.data_ptr()), ctypes.c_size_t(N * 8), 2)
    dt = time.perf_counter() - t0
print(f"D2H int64 into registered buffer: {N*8/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cudart.cudaMemcpy(ctypes.c_void_p(host.ctypes.data), ctypes.c_void_p(dev32.data_ptr()), ctypes.c_size_t(N * 4), 2)
    dt = time.perf_counter() - t0
print(f"D2H int32 (half) into registered buffer: {N*4/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)")
cudart.cudaHostUnregister(ctypes.c_void_p(host.ctypes.data))
# host write bandwidth: numpy fill with threads
from concurrent.futures import ThreadPoolExecutor
def fill(t, T=16):
    a, b = N * t // T, N * (t + 1) // T
    host[a:b] = 7
for T in (8, 16):
    with ThreadPoolExecutor(T) as ex:
        for _ in range(3):
            t0 = time.perf_counter(); list(ex.map(lambda t: fill(t, T), range(T))); dt = time.perf_counter() - t0
    print(f"host fill {T} threads: {N*8/dt/1e9:.1f} GB/s")
