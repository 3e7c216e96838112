"""A/B the public-build e2e under bench-like conditions (diagnostic)."""
import os, sys, statistics, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_06713_b200 as b200
from paper_2401_06713_b200 import _native
from paper_2401_06713_b200.conflict import stage
import bench

view, lists, _ = bench.make_inputs("c2", pinned=True)
ctx = _native.context(0)

def e2e(tag):
    ts = []
    for k in range(8):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        g = b200.build(view, lists)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0); g = None
    print(f"{tag}: median {statistics.median(ts[2:])*1e3:.2f} ms  all {[round(t*1e3,1) for t in ts]}", flush=True)

e2e("fresh process")
ctx.profiling(True)
e2e("profiling on")
ctx.profiling(False)
stage(view, lists, ctx)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(10):
    ctx.build_device()
e2e("after device loop")
ctx.profiling(True)
for _ in range(10):
    ctx.build_device()
e2e("after device loop, profiling on")
