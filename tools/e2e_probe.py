"""Break the public build() e2e time into its phases on one GPU (diagnostic, not a bench)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2401_06713_b200 as b200
from paper_2401_06713_b200 import conflict, _native
import bench

view, lists, _ = bench.make_inputs(sys.argv[1] if len(sys.argv) > 1 else "c2", pinned=True)
n = view.n_active
for rep in range(4):
    t = [time.perf_counter()]
    ctx = conflict.stage(view, lists); torch.cuda.synchronize(); t.append(time.perf_counter())
    c = ctx.count(0, 1, 0, n); t.append(time.perf_counter())
    total = c.deg_sum // 2; nm = c.members_in_range
    members = np.empty(nm, dtype=np.int64); offsets = np.empty(nm + 1, dtype=np.int64)
    neighbors = np.empty(2 * total, dtype=np.int64); t.append(time.perf_counter())
    ctx.fill(members, offsets, neighbors); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"stage {d[0]:.2f} count {d[1]:.2f} alloc {d[2]:.2f} fill+d2h {d[3]:.2f} total {sum(d):.2f} ms")
# raw link + host write speeds
nb = 2 * total * 4
dev = torch.empty(nb // 4, dtype=torch.int32, device="cuda")
pin = torch.empty(nb // 4, dtype=torch.int32, pin_memory=True)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); pin.copy_(dev); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"D2H pinned {nb/dt/1e9:.1f} GB/s ({nb/1e6:.0f} MB in {dt*1e3:.1f} ms)")
src = pin.numpy()
for _ in range(3):
    t0 = time.perf_counter(); out = np.empty(src.size, np.int64); out[:] = src; dt = time.perf_counter() - t0
print(f"host widen into fresh array (numpy 1 thread) {dt*1e3:.1f} ms")
for _ in range(3):
    t0 = time.perf_counter(); out[:] = src; dt = time.perf_counter() - t0
print(f"host widen into touched array {dt*1e3:.1f} ms")
print("cores", os.cpu_count(), "omp", os.environ.get("OMP_NUM_THREADS"))

def timed_fill(make):
    ts = []
    for _ in range(3):
        ctx = conflict.stage(view, lists); c = ctx.count(0, 1, 0, n)
        total = c.deg_sum // 2; nm = c.members_in_range
        t0 = time.perf_counter()
        members, offsets, neighbors = make(nm), make(nm + 1), make(2 * total)
        ctx.fill(members, offsets, neighbors)
        ts.append((time.perf_counter() - t0) * 1e3)
        del members, offsets, neighbors
    return " ".join(f"{x:.1f}" for x in ts)

pool = {}
def touched(k):
    a = pool.get(k)
    if a is None:
        a = pool[k] = np.ones(k, np.int64)
    return a
print("fill into fresh numpy   ", timed_fill(lambda k: np.empty(k, np.int64)))
print("fill into touched numpy ", timed_fill(touched))
print("fill into torch pinned  ", timed_fill(lambda k: torch.empty(k, dtype=torch.int64, pin_memory=True).numpy()))
dev64 = torch.empty(2 * total, dtype=torch.int64, device="cuda")
pin64 = torch.empty(2 * total, dtype=torch.int64, pin_memory=True)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); pin64.copy_(dev64); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"D2H int64 into pinned {2*total*8/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)")
import ctypes
from paper_2401_06713_b200 import _native as nat
# multi-thread host widening speed via numpy in threads
from concurrent.futures import ThreadPoolExecutor
src32 = pin.numpy(); dst = pool[2 * total]
def part(t, T=16):
    a, b = src32.size * t // T, src32.size * (t + 1) // T
    dst[a:b] = src32[a:b]
with ThreadPoolExecutor(16) as ex:
    for _ in range(3):
        t0 = time.perf_counter(); list(ex.map(part, range(16))); dt = time.perf_counter() - t0
print(f"16-thread numpy widen into touched {dt*1e3:.1f} ms")
print("public build() steady state with the host pool:")
for _ in range(4):
    t0 = time.perf_counter(); g = b200.build(view, lists); dt = time.perf_counter() - t0; g = None
    print(f"  {dt*1e3:.1f} ms")
