"""Public-API build() steady-state time at config 2 for D2H pipeline settings (diagnostic)."""
import os, sys, statistics, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_06713_b200 as b200
from paper_2401_06713_b200 import _native
import bench

view, lists, _ = bench.make_inputs("c2", pinned=True)
ctx = _native.context()
configs = [(1 << 20, 16, 0), (1 << 19, 16, 0), (1 << 21, 16, 0), (1 << 20, 8, 0), (1 << 22, 16, 0), (1 << 20, 16, 4)]
for ch, thr, mode in configs:
    ring = mode
    ctx.option("d2h_chunk", ch); ctx.option("d2h_threads", thr); ctx.option("d2h_mode", mode)
    ts = []
    for k in range(7):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        g = b200.build(view, lists)
        ts.append(time.perf_counter() - t0); g = None
    print(f"chunk {ch:>8} ids mode {ring:2d} threads {thr:2d}: median {statistics.median(ts[2:])*1e3:6.1f} ms  min {min(ts[2:])*1e3:6.1f}", flush=True)

ctx.option("d2h_mode", 0)
# phases of one public build
from paper_2401_06713_b200 import conflict
import numpy as np
n = view.n_active
for rep in range(3):
    t = [time.perf_counter()]
    c = conflict.stage(view, lists, ctx); torch.cuda.synchronize(); t.append(time.perf_counter())
    cc = ctx.count(0, 1, 0, n); t.append(time.perf_counter())
    total = cc.deg_sum // 2; nm = cc.members_in_range
    from paper_2401_06713_b200 import hostpool
    members = np.empty(nm, dtype=np.int64); offsets = np.empty(nm + 1, dtype=np.int64)
    neighbors = hostpool.empty_int64(2 * total); t.append(time.perf_counter())
    ctx.fill(members, offsets, neighbors); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"stage+prep {d[0]:.2f} count {d[1]:.2f} alloc {d[2]:.2f} fill+d2h {d[3]:.2f} total {sum(d):.2f} ms", flush=True)
    neighbors = None
