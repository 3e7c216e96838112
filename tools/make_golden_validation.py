"""Golden validation reports from the REFERENCE validator (validation.py:41-131).

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden_validation.py

For a few Pauli instances: a proper coloring (a whole reference run) and deliberately broken
colorings (merged color classes, one recolored vertex, an uncolored vertex), each on the full
view and on an induced subset.  Stores the inputs needed to rebuild them (generator args and
the color arrays) and the reference's report fields -> tests/golden/validation.npz + .json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import palettecolor as pc  # noqa: E402  (the reference)
from palettecolor import validation  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
arrays, index = {}, []


def add(name, n, q, gseed, color, active=None, note=""):
    ps = pc.PauliSet.from_strings(pc.random_pauli_strings(n, q, seed=gseed))
    view = pc.pauli_view(ps) if active is None else pc.pauli_view(ps).induce(np.asarray(active))
    res = pc.run(pc.pauli_view(ps), pc.PaletteParams(12.5, 2.0, seed=0))
    res.color = np.asarray(color, dtype=np.int64)  # the report reads color + iterations only
    rep = validation.validate(view, res, "exhaustive")
    arrays[f"{name}/color"] = res.color
    if active is not None:
        arrays[f"{name}/active"] = np.asarray(active, dtype=np.int64)
    index.append({"name": name, "n": n, "q": q, "gen_seed": gseed, "note": note,
                  "subset": active is not None,
                  "proper": rep.proper, "violation_count": rep.violation_count,
                  "violations": [list(map(int, p)) for p in rep.violations],
                  "colors_used": rep.colors_used, "oracle_edges": rep.oracle_edges,
                  "pairs_checked": rep.pairs_checked, "ec_max_pct": rep.ec_max_pct})
    print(name, rep.proper, rep.violation_count, rep.oracle_edges)


for n, q, gseed in [(300, 8, 1), (2000, 16, 0), (5000, 32, 3)]:
    ps = pc.PauliSet.from_strings(pc.random_pauli_strings(n, q, seed=gseed))
    res = pc.run(pc.pauli_view(ps), pc.PaletteParams(12.5, 2.0, seed=0))
    good = res.color.copy()
    add(f"n{n}_proper", n, q, gseed, good, note="reference run, proper")
    rng = np.random.default_rng(gseed)
    merged = good.copy()
    a, b = np.unique(good)[:2]
    merged[merged == b] = a
    add(f"n{n}_merged", n, q, gseed, merged, note="two color classes merged")
    few = good.copy()
    few[:] = good % 5  # many violations: sample cap, order
    add(f"n{n}_mod5", n, q, gseed, few, note="colors mod 5: thousands of violations")
    unc = few.copy()
    unc[rng.choice(n, n // 3, replace=False)] = pc.UNCOLORED
    add(f"n{n}_uncolored", n, q, gseed, unc, note="a third uncolored (never a violation)")
    sub = np.sort(rng.choice(n, n // 2, replace=False))
    add(f"n{n}_mod5_subset", n, q, gseed, few, active=sub, note="induced half")

np.savez_compressed(os.path.join(OUT, "validation.npz"), **arrays)
with open(os.path.join(OUT, "validation.json"), "w") as f:
    json.dump(index, f, indent=1)
