"""e2e median per worker-thread count, interleaved rounds (diagnostic)."""
import os, sys, statistics, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_06713_b200 as b200
from paper_2401_06713_b200 import _native
import bench

view, lists, _ = bench.make_inputs("c2", pinned=True)
ctx = _native.context(0)
res = {}
for rnd in range(3):
    for W in (8, 10, 12, 14, 15, 16):
        ctx.option("d2h_threads", W)
        ts = []
        for k in range(6):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            g = b200.build(view, lists)
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t0); g = None
        res.setdefault(W, []).append(statistics.median(ts[1:]) * 1e3)
for W, v in res.items():
    print(W, [round(x, 2) for x in v], flush=True)
print("OMP_PROC_BIND", os.environ.get("OMP_PROC_BIND"), "nproc", os.cpu_count())
