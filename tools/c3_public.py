"""Config 3 through the public build (e2e) with sanity checks (diagnostic): sortedness,
no self loops, offsets/size consistency, symmetry of sampled rows.  The oracle comparison of
sampled rows is tests/test_gpu_scale.py (PICASSO_SCALE=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2401_06713_b200 as b200
import bench

view, lists, plan = bench.make_inputs("c3", pinned=True)
n = view.n_active
for k in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    gc = b200.build(view, lists)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"public build c3: {dt*1e3:.1f} ms  |E_c|={gc.edge_count} |E|={gc.view_edges_scanned} "
          f"pairs/s={n*(n-1)/2/dt:.3e}", flush=True)
    if k < 2:
        gc = None
off, nb = gc.graph.offsets, gc.graph.neighbors
assert off[-1] == nb.size == 2 * gc.edge_count
rng = np.random.default_rng(0)
rows = rng.choice(gc.members.size, 24, replace=False)
for r in rows:
    row = nb[off[r]:off[r + 1]]
    assert np.all(np.diff(row) > 0) and not np.any(row == r)
    for j in row[:5]:
        rj = nb[off[j]:off[j + 1]]
        assert r in rj
print("c3 sampled rows: sorted, symmetric, consistent")
