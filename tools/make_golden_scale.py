"""Full-size goldens from the scale oracle (oracle/bucket_oracle.c) -> tests/golden/scale.json.

The reference cannot run at configs 2-4 (O(n^2) index arrays, a 250 GB palette
mask at config 4), so these hashes come from the scale oracle, which tests/test_scale_oracle.py
pins against the reference's own outputs (every golden build, the q=32 5k/10k/20k hashes,
the c1 per-iteration hashes) and against the dense-mask oracle.  This script additionally
re-derives the reference's recorded 50k whole run (7,498 colors, color sha
5acbe96d9c45c44b) before writing anything, so a whole run driven by the scale oracle is
pinned against the reference at 25x the c1 size.

    python tools/make_golden_scale.py --builds c2 c3 c4 --runs c2 c3

Hashes: oracle/scale.py csr_hashes (members/offsets sha16, block hash of the int64
neighbors).  The GPU tests (tests/test_gpu_full_parity.py) hash the product's output the same way.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2401_06713_b200 as b200  # noqa: E402
from oracle.scale import ScaleOracle, csr_hashes, sha16  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "scale.json")
CONFIGS = {  # name: (n, q, gen_seed, palette_pct, alpha, seed)
    "c2": (100_000, 32, 0, 12.5, 2.0, 0),
    "c3": (1_000_000, 64, 0, 12.5, 2.0, 0),
    "c4": (4_000_000, 128, 0, 12.5, 2.0, 0),
    "q32_n50000": (50_000, 32, 0, 12.5, 2.0, 0),
    # config 5 grid cells (500k x 64q, palette P' and alpha varied)
    "c5_p20_a0.5": (500_000, 64, 0, 20.0, 0.5, 0),
    "c5_p5_a2": (500_000, 64, 0, 5.0, 2.0, 0),
    "c5_p2.5_a3": (500_000, 64, 0, 2.5, 3.0, 0),
}


def inputs(name):
    n, q, gseed, pct, alpha, seed = CONFIGS[name]
    ps = b200.PauliSet.from_strings(b200.random_pauli_strings(n, q, seed=gseed))
    view = b200.pauli_view(ps)
    params = b200.PaletteParams(pct, alpha, seed=seed)
    return view, params


def oracle_builder(trace):
    from paper_2401_06713_b200.conflict import ConflictGraph
    from paper_2401_06713_b200.graph import ExplicitGraph

    def build(view, lists, **kw):
        t = time.time()
        o = ScaleOracle(view.backing.words, view.active, lists)
        r = o.build()
        o.close()
        h = csr_hashes(r.members, r.offsets, r.neighbors, r.edge_count, r.view_edges_scanned)
        h.update(n_active=int(view.n_active), active_sha=sha16(view.active),
                 lists_sha=sha16(lists.array), palette_base=int(lists.palette_base),
                 palette_size=int(lists.palette_size))
        trace.append(h)
        print(f"  build n={view.n_active} |E_c|={r.edge_count} {time.time() - t:.1f}s", flush=True)
        return ConflictGraph(r.members, ExplicitGraph(int(r.members.size), r.offsets, r.neighbors),
                             r.edge_count, r.view_edges_scanned)

    return build


def golden_build(name):
    view, params = inputs(name)
    n = view.n_active
    plan = b200.plan_iteration(1, n, params)
    lists = b200.assign_random_lists(plan, view.active, params.seed, device=False)
    t = time.time()
    o = ScaleOracle(view.backing.words, view.active, lists)
    h = o.hashes()
    o.close()
    h.update(n=n, q=CONFIGS[name][1], words_sha=sha16(view.backing.words.view(np.int64)),
             lists_sha=sha16(lists.array), palette_size=plan.palette_size,
             list_size=plan.list_size, oracle_seconds=round(time.time() - t, 1))
    print(name, h, flush=True)
    return h


def golden_run(name):
    view, params = inputs(name)
    trace = []
    t = time.time()
    res = b200.run(view, params, builder=oracle_builder(trace))
    out = dict(n=view.n_active, q=CONFIGS[name][1], colors=int(res.total_colors),
               iterations=len(res.iterations), oracle_edges=int(res.oracle_edges),
               peak_conflict_edges=int(res.peak_conflict_edges), color_sha=sha16(res.color),
               colored_at_sha=sha16(res.colored_at), builds=trace,
               records=[dict(n_active=r.n_active, palette_size=r.palette_size,
                             list_size=r.list_size, conflict_vertices=r.conflict_vertices,
                             conflict_edges=r.conflict_edges,
                             colored_in_conflict=r.colored_in_conflict, uncolored=r.uncolored)
                        for r in res.iterations],
               oracle_seconds=round(time.time() - t, 1))
    print(name, {k: v for k, v in out.items() if k not in ("builds", "records")}, flush=True)
    return out


def golden_run_counts(name):
    """A whole run whose builds are the oracle's counts only (members, offsets, edge counts:
    bucket_oracle.c degrees) and whose coloring is the word-predicate list coloring — the
    form of driver.run(conflict_rows=False), for configs whose per-iteration CSR does not fit
    this host (config 4: 115 GB at iteration 1).  Iteration 1's view_edges_scanned is taken
    from the config's build golden when present (its commute count alone is ~1.5 h here)."""
    from paper_2401_06713_b200 import list_coloring
    from paper_2401_06713_b200.conflict import ConflictGraph
    from paper_2401_06713_b200.graph import ExplicitGraph

    view, params = inputs(name)
    known = json.load(open(OUT))["builds"].get(name, {}) if os.path.exists(OUT) else {}
    trace = []

    def counts_builder(v, lists, **kw):
        t = time.time()
        o = ScaleOracle(v.backing.words, v.active, lists)
        deg, _ = o.degrees()
        has = deg > 0
        members = np.asarray(v.active, dtype=np.int64)[has]
        offsets = np.zeros(members.size + 1, dtype=np.int64)
        np.cumsum(deg[has], out=offsets[1:])
        first = not trace
        if first and known.get("lists_sha") == sha16(lists.array):
            scanned = int(known["view_edges_scanned"])
        else:
            scanned = o.commute_count()
        o.close()
        h = dict(n_active=int(v.n_active), active_sha=sha16(v.active), lists_sha=sha16(lists.array),
                 members_sha=sha16(members), offsets_sha=sha16(offsets), n_members=int(members.size),
                 edge_count=int(deg.sum()) // 2, view_edges_scanned=scanned)
        trace.append(h)
        print(f"  counts n={v.n_active} |E_c|={h['edge_count']} {time.time() - t:.1f}s", flush=True)
        return ConflictGraph(members, ExplicitGraph(int(members.size), offsets, np.zeros(0, np.int64)),
                             h["edge_count"], scanned)

    t = time.time()
    # (the driver hands each iteration's view to the coloring: word-predicate adjacency)
    res = b200.run(view, params, builder=counts_builder,
                   conflict_coloring=list_coloring.color_conflict_graph)
    out = dict(n=view.n_active, q=CONFIGS[name][1], colors=int(res.total_colors),
               iterations=len(res.iterations), oracle_edges=int(res.oracle_edges),
               peak_conflict_edges=int(res.peak_conflict_edges), color_sha=sha16(res.color),
               colored_at_sha=sha16(res.colored_at), builds=trace,
               records=[dict(n_active=r.n_active, palette_size=r.palette_size,
                             list_size=r.list_size, conflict_vertices=r.conflict_vertices,
                             conflict_edges=r.conflict_edges,
                             colored_in_conflict=r.colored_in_conflict, uncolored=r.uncolored)
                        for r in res.iterations],
               counts_only=True, oracle_seconds=round(time.time() - t, 1))
    print(name, {k: v for k, v in out.items() if k not in ("builds", "records")}, flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--builds", nargs="*", default=[])
    ap.add_argument("--runs", nargs="*", default=[])
    ap.add_argument("--skip-pin", action="store_true")
    ap.add_argument("--runs-counts", nargs="*", default=[],
                    help="whole runs in the counts-only form (driver.run(conflict_rows=False))")
    a = ap.parse_args()
    with open(os.path.join(ROOT, "tests", "golden", "reference.json")) as f:
        rec = json.load(f)["runs_recorded"]["q32_n50000"]
    gold = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            gold = json.load(f)
    gold.setdefault("builds", {})
    gold.setdefault("runs", {})
    if not a.skip_pin:
        r = golden_run("q32_n50000")
        for k in ("colors", "iterations", "oracle_edges", "peak_conflict_edges", "color_sha"):
            assert r[k] == rec[k], (k, r[k], rec[k])
        print("q32_n50000 whole run equals the reference's recorded run", flush=True)
        gold["runs"]["q32_n50000"] = r
    for name in a.builds:
        gold["builds"][name] = golden_build(name)
        with open(OUT, "w") as f:
            json.dump(gold, f, indent=1)
    for name in a.runs:
        gold["runs"][name] = golden_run(name)
        with open(OUT, "w") as f:
            json.dump(gold, f, indent=1)
    for name in a.runs_counts:
        r = golden_run_counts(name)
        with open(OUT) as f:  # (other writers may have added entries meanwhile)
            gold = json.load(f)
        gold.setdefault("runs_counts", {})[name] = r
        with open(OUT, "w") as f:
            json.dump(gold, f, indent=1)
    with open(OUT, "w") as f:
        json.dump(gold, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
