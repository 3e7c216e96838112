"""A whole Picasso run (driver.run: GPU builds, GPU palette lists, native list coloring) on
config 3 (1M x 64q), with the per-iteration table (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_06713_b200 as b200

n, q = 1_000_000, 64
t0 = time.time()
view = b200.pauli_view(b200.PauliSet.from_strings(b200.random_pauli_strings(n, q, seed=0)))
print(f"inputs {time.time() - t0:.1f} s", flush=True)
t0 = time.time()
res = b200.run(view, b200.PaletteParams(12.5, 2.0, seed=0))
wall = time.time() - t0
cols = res.color[res.color >= 0]
print(f"c3 whole run: {wall:.1f} s, {len(res.iterations)} iterations, {len(set(cols.tolist()))} colors, "
      f"completed={res.completed}", flush=True)
for r in res.iterations:
    d = r.__dict__ if hasattr(r, "__dict__") else r._asdict()
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items()})

# exhaustive properness check of the coloring on the GPU (the reference's validator stops at
# 20,000 vertices): every commuting pair with equal colors is a violation
from paper_2401_06713_b200.validation import validate

t0 = time.time()
rep = validate(view, res, "exhaustive", uncapped=True)
print(f"validate (exhaustive, GPU): proper={rep.proper} violations={rep.violation_count} "
      f"colors={rep.colors_used} |E|={rep.oracle_edges} in {time.time() - t0:.2f} s", flush=True)
