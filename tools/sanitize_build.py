"""One public build under compute-sanitizer (evidence run, not a test): the default kernels
(prep, owned masks, K1, count, fill, copy-out) on a small instance, checked against the scale
oracle.  Usage: compute-sanitizer --tool <memcheck|racecheck|synccheck|initcheck>
python tools/sanitize_build.py N Q [fill_algo [own_direct]]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2401_06713_b200 as b200  # noqa: E402
from paper_2401_06713_b200 import _native  # noqa: E402
from oracle.scale import scale_build  # noqa: E402

n, q = int(sys.argv[1]), int(sys.argv[2])
fill = int(sys.argv[3]) if len(sys.argv) > 3 else 0
own_direct = int(sys.argv[4]) if len(sys.argv) > 4 else 1  # 0: the bitmap ownership at small P
v = b200.pauli_view(b200.PauliSet.from_strings(b200.random_pauli_strings(n, q, seed=0)))
plan = b200.plan_iteration(1, n, b200.PaletteParams(12.5, 2.0, seed=0))
lists = b200.assign_random_lists(plan, v.active, 0, device=False)
_native.context().option("fill_algo", fill)
_native.context().option("own_direct", own_direct)
gc = b200.build(v, lists)
want = scale_build(v, lists)
ok = (np.array_equal(gc.members, want.members) and np.array_equal(gc.graph.offsets, want.offsets)
      and np.array_equal(gc.graph.neighbors, want.neighbors)
      and gc.view_edges_scanned == want.view_edges_scanned)
print(f"sanitized build n={n} q={q} fill_algo={fill} own_direct={own_direct}: |E_c|={gc.edge_count} parity={'OK' if ok else 'MISMATCH'}")
sys.exit(0 if ok else 1)
