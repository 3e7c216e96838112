"""Quick device timing of one build configuration (development aid, not the bench)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time

import numpy as np

import paper_2401_06713_b200 as b200
from paper_2401_06713_b200 import _native
from paper_2401_06713_b200.conflict import stage

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--q", type=int, default=32)
ap.add_argument("--algo", type=int, default=0)
ap.add_argument("--window", type=int, default=0)
ap.add_argument("--k2", type=int, default=0)
ap.add_argument("--fill", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--seg-bits", type=int, default=0)
ap.add_argument("--seg-warps", type=int, default=0)
ap.add_argument("--own", type=int, default=0)
ap.add_argument("--own-direct", type=int, default=1)
ap.add_argument("--blk-threads", type=int, default=0)
ap.add_argument("--blk-groups", type=int, default=0)
ap.add_argument("--blk-ecap", type=int, default=0)
ap.add_argument("--blk-dcap", type=int, default=0)
ap.add_argument("--bins-threads", type=int, default=0)
ap.add_argument("--bins-shift", type=int, default=0)
ap.add_argument("--bins-maxdeg", type=int, default=0)
ap.add_argument("--async", dest="k1_async", type=int, default=0)
ap.add_argument("--early", type=int, default=2)
ap.add_argument("--check", action="store_true", help="compare the CSR with the default fill")
ap.add_argument("--pct", type=float, default=12.5)
ap.add_argument("--ichunk", type=int, default=0)
ap.add_argument("--k1-warps", type=int, default=0)
ap.add_argument("--dyn", type=int, default=1)
ap.add_argument("--own-bitmap", type=int, default=1)
ap.add_argument("--alpha", type=float, default=2.0)
a = ap.parse_args()

t = time.time()
v = b200.pauli_view(b200.PauliSet.from_strings(b200.random_pauli_strings(a.n, a.q, seed=0)))
plan = b200.plan_iteration(1, a.n, b200.PaletteParams(a.pct, a.alpha, seed=0))
lists = b200.assign_random_lists(plan, v.active, 0)
print(f"inputs {time.time()-t:.1f}s  P={plan.palette_size} L={plan.list_size}", flush=True)
ctx = _native.context()
ctx.option("k1_algo", a.algo)
ctx.option("window", a.window)
ctx.option("k2_mode", a.k2)
ctx.option("fill_algo", a.fill)
ctx.option("seg_bits", a.seg_bits)
ctx.option("seg_warps", a.seg_warps)
ctx.option("own_algo", a.own)
ctx.option("own_direct", a.own_direct)
ctx.option("blk_threads", a.blk_threads)
ctx.option("blk_groups", a.blk_groups)
ctx.option("blk_ecap", a.blk_ecap)
ctx.option("blk_dcap", a.blk_dcap)
ctx.option("bins_threads", a.bins_threads)
ctx.option("bins_shift", a.bins_shift)
ctx.option("bins_maxdeg", a.bins_maxdeg)
ctx.option("k1_async", a.k1_async)
ctx.option("k1_early", a.early)
ctx.option("fr_ichunk", a.ichunk)
ctx.option("k1_warps", a.k1_warps)
ctx.option("dyn_work", a.dyn)
ctx.option("own_bitmap", a.own_bitmap)
ctx.profiling(True)
stage(v, lists, ctx)
print("prep ms", ctx.kernel_times()[4])
pairs = a.n * (a.n - 1) // 2
import torch  # noqa: E402  (events only)

for r in range(a.reps):
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    c, nl = ctx.build_device()
    t1.record()
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    print(f"rep {r}: total {t0.elapsed_time(t1):.3f} ms  prep {kt[4]:.3f}  K1 {kt[0]:.3f} ms ({pairs/kt[0]/1e9:.1f} Gpair/s)  "
          f"K2count {kt[1]:.3f}  compact {kt[3]:.3f}  K2fill {kt[2]:.3f}  launches {nl}  "
          f"|E_c|={c.deg_sum//2} |E|={c.pairs_in_shard-c.anticommuting}", flush=True)
t = time.time()
gc = b200.build(v, lists)
print(f"e2e build {time.time()-t:.3f} s")
if a.check:  # the same CSR with the default fill
    import hashlib
    h = lambda x: hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()[:16]
    got = (h(gc.graph.offsets), h(gc.graph.neighbors), h(gc.members))
    gc = None
    ctx.option("fill_algo", 0)
    ref = b200.build(v, lists)
    want = (h(ref.graph.offsets), h(ref.graph.neighbors), h(ref.members))
    print("check vs default fill:", "MATCH" if got == want else f"MISMATCH {got} {want}")
