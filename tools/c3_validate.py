"""Config-3 whole run validated exhaustively on the GPU (evidence run, not a test).

The run (GPU builds, GPU palette lists, native list coloring) is checked against the golden
coloring (tests/golden/scale.json: color sha from the oracle-driven run), then every pair
inside every color class is checked with the commute predicate on the GPU (validation.validate,
uncapped: the reference stops at 20,000 vertices) — a check independent of the conflict CSR.
Usage: python tools/c3_validate.py > profiles/r2_c3_validation.txt
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2401_06713_b200 as b200  # noqa: E402
from paper_2401_06713_b200 import validation  # noqa: E402

view = b200.pauli_view(b200.PauliSet.from_strings(b200.random_pauli_strings(1_000_000, 64, seed=0)))
t = time.perf_counter()
res = b200.run(view, b200.PaletteParams(12.5, 2.0, seed=0))
t_run = time.perf_counter() - t
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "scale.json")))["runs"]["c3"]
sha = hashlib.sha256(np.ascontiguousarray(res.color, dtype=np.int64).data).hexdigest()[:16]
print(f"c3 whole run: {t_run:.2f} s, {res.total_colors} colors, {len(res.iterations)} iterations, "
      f"color sha {sha} (golden {gold['color_sha']}: {'identical' if sha == gold['color_sha'] else 'DIFFERENT'})")
t = time.perf_counter()
rep = validation.validate(view, res, uncapped=True)
t_val = time.perf_counter() - t
print(f"exhaustive validation (GPU, uncapped): {t_val:.2f} s; proper={rep.proper} "
      f"violations={rep.violation_count} colors_used={rep.colors_used} "
      f"oracle_edges={rep.oracle_edges} (run: {res.oracle_edges})")
ok = sha == gold["color_sha"] and rep.proper and rep.violation_count == 0 and rep.oracle_edges == res.oracle_edges
print("OK" if ok else "FAILED")
sys.exit(0 if ok else 1)
