"""A/B of the pipelined public fill (d2h_pipe 1) against fill-then-copy-out (d2h_pipe 0),
interleaved in one process on the same inputs (diagnostic)."""
import os, sys, statistics, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_06713_b200 as b200
from paper_2401_06713_b200 import _native
import bench

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
view, lists, _ = bench.make_inputs(wl, pinned=True)
ctx = _native.context(0)
res = {}
# configs: pipe:pieces:threads[:dma%] tokens, e.g. 0:0:16 1:8:0:25
specs = sys.argv[2:] or ["0:0:16", "1:6:16", "1:6:15", "1:12:15", "1:4:15", "1:8:15"]
configs = [(sp, *(list(map(int, sp.split(":"))) + [-1])[:4]) for sp in specs]
for rnd in range(6):
    for tag, pipe, pieces, thr, dma in configs:
        ctx.option("d2h_pipe", pipe)
        ctx.option("d2h_pieces", pieces)
        ctx.option("d2h_threads", thr)
        ctx.option("d2h_dma", dma)
        for k in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            g = b200.build(view, lists)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0; g = None
            if rnd > 0 or k > 0:
                res.setdefault(tag, []).append(dt * 1e3)
for tag, *_ in configs:
    v = res[tag]
    print(f"{tag}: median {statistics.median(v):.2f} ms  min {min(v):.2f}  n={len(v)}", flush=True)
