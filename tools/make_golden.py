"""Generate tests/golden/* by running the REFERENCE package (read-only, imported here).

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py

Outputs (all committed):
  tests/golden/builds_small.npz  — full inputs + reference CSR for small Pauli builds
                                   (test_conflict.py Pauli cases, acceptance-4 Pauli cases,
                                   induced residue views, a ragged-list view, edge cases)
  tests/golden/reference.json    — known-answer vectors (encoding, RNG) and SHA-256 prefixes
                                   of the reference CSR for larger builds and whole runs
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import palettecolor as pc  # noqa: E402  (the reference)
from palettecolor import conflict, rng  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()[:16]


def u64hex(a) -> list[str]:
    return [f"0x{int(x):016x}" for x in np.asarray(a, dtype=np.uint64).ravel()]


cases: dict[str, np.ndarray] = {}
index: list[dict] = []


def add_case(name, view, lists, note):
    ref = conflict.build(view, lists)
    naive = conflict.build_reference(view, lists) if view.n_active <= 400 else None
    if naive is not None:
        assert np.array_equal(naive.graph.neighbors, ref.graph.neighbors)
    words = view.backing.words
    cases[f"{name}/words"] = np.asarray(words, dtype=np.uint64)
    cases[f"{name}/active"] = view.active.astype(np.int64)
    if lists.array is not None:
        cases[f"{name}/lists"] = lists.array.astype(np.int64)
    else:
        cases[f"{name}/list_data"] = np.concatenate(lists.rows).astype(np.int64)
        cases[f"{name}/list_off"] = np.concatenate(
            [[0], np.cumsum([r.size for r in lists.rows])]
        ).astype(np.int64)
    cases[f"{name}/members"] = ref.members.astype(np.int64)
    cases[f"{name}/offsets"] = ref.graph.offsets.astype(np.int64)
    cases[f"{name}/neighbors"] = ref.graph.neighbors.astype(np.int32)
    index.append(
        dict(
            name=name,
            note=note,
            num_qubits=int(view.backing.num_qubits),
            n_total=int(view.backing.n),
            n_active=int(view.n_active),
            palette_base=int(lists.palette_base),
            palette_size=int(lists.palette_size),
            edge_count=int(ref.edge_count),
            view_edges_scanned=int(ref.view_edges_scanned),
        )
    )


def pauli_view(n, q, seed):
    ps = pc.PauliSet.from_strings(pc.random_pauli_strings(n, q, seed=seed))
    return pc.pauli_view(ps)


def random_lists(view, pct=12.5, alpha=2.0, seed=0, iteration=1, base=0):
    plan = pc.plan_iteration(iteration, view.n_active, pc.PaletteParams(pct, alpha, seed), palette_base=base)
    return pc.assign_random_lists(plan, view.active, seed)


def main():
    os.makedirs(OUT, exist_ok=True)
    # test_conflict.py Pauli cases
    v = pauli_view(120, 5, 4)
    add_case("tc_all_modes_pauli", v, random_lists(v, seed=2), "test_conflict.py:95-102")
    v = pauli_view(150, 6, 9)
    add_case("tc_determinism", v, random_lists(v, seed=7), "test_conflict.py:112-121")
    v = pauli_view(60, 5, 2)
    add_case("tc_csr_invariants", v, random_lists(v, seed=5), "test_conflict.py:150-158")
    # acceptance criterion 4, Pauli instances (every 3rd k)
    for k in range(0, 30, 3):
        n = 20 + k * 16
        v = pauli_view(n, 4 + k % 6, k)
        plan = pc.plan_iteration(1, n, pc.PaletteParams(10.0 + (k % 4) * 5, 1.0 + (k % 3), seed=k))
        add_case(f"acc4_k{k}", v, pc.assign_random_lists(plan, v.active, seed=k), "test_acceptance.py:139-158")
    # induced residue view (iteration 2 palette on a subset)
    v = pauli_view(600, 7, 11)
    sub = v.induce(np.arange(3, 600, 3))
    add_case("induced_subset", sub, random_lists(sub, seed=3, iteration=2, base=75), "graph.py:357-366")
    # ragged lists on a Pauli view (ColorLists.from_dict)
    v = pauli_view(90, 6, 5)
    r = np.random.default_rng(17)
    d = {int(i): sorted(set(r.integers(0, 40, size=int(r.integers(1, 9))).tolist())) for i in range(90)}
    add_case("ragged_lists", v, pc.ColorLists.from_dict(d), "driver.py:120-135")
    # single-color palette: every commuting pair conflicts
    v = pauli_view(40, 3, 8)
    plan = pc.IterationPlan(iteration=1, palette_size=1, palette_base=9, list_size=1)
    add_case("single_color", v, pc.assign_random_lists(plan, v.active, 0), "driver.py:61-86")
    # duplicates / identities: q=1 gives many identical strings
    v = pauli_view(50, 1, 3)
    add_case("q1_duplicates", v, random_lists(v, pct=30, seed=1), "pauli.py:194-203")
    # word-boundary qubit counts (21, 22, 43 qubits -> 63/66/129 bits)
    for q in (21, 22, 43, 65):
        v = pauli_view(200, q, q)
        add_case(f"q{q}_boundary", v, random_lists(v, seed=q), "pauli.py:7-14")
    # a view with two vertices and no conflicts possible
    v = pauli_view(2, 4, 0)
    add_case("two_vertices", v, pc.ColorLists.from_dict({0: [0], 1: [1]}), "conflict.py:150,158")
    # full c1 iteration-1 build stored in full (n=2000)
    v = pauli_view(2000, 16, 0)
    add_case("c1_iter1", v, random_lists(v, seed=0), "BASELINE config 1, iteration 1")

    np.savez_compressed(os.path.join(OUT, "builds_small.npz"), **cases)

    ref = {"cases": index}
    # ---- encoding known answers
    strings = pc.random_pauli_strings(2000, 16, seed=0)
    ref["encode"] = {
        "c1_first3": strings[:3],
        "c1_words_first3": u64hex(pc.PauliSet.from_strings(strings[:3]).words[:, 0]),
        "XYZI": int(pc.encode("XYZI").value),
        "q22_words": u64hex(pc.PauliSet.from_strings(["XYZI" * 5 + "YZ"]).words),
        "gen_hash": {
            f"{n}x{q}s{s}": hashlib.sha256("\n".join(pc.random_pauli_strings(n, q, seed=s)).encode()).hexdigest()[:16]
            for (n, q, s) in [(2000, 16, 0), (1000, 11, 1000), (300, 8, 3), (500, 64, 7)]
        },
        "gen_exclude_identity": pc.random_pauli_strings(8, 1, seed=2, exclude_identity=True),
    }
    # ---- RNG known answers (rng.py has no known-answer test of its own)
    keys = rng.stream_keys(0, 1, [0, 1, 2])
    ref["rng"] = {
        "mix64_0_1_2": u64hex(rng.mix64(np.array([0, 1, 2], dtype=np.uint64))),
        "stream_keys_0_1": u64hex(keys),
        "stream_keys_neg": u64hex(rng.stream_keys(-5, 3, [0, 7, 1 << 40])),
        "sample_250_15_row0": rng.sample_distinct(keys, 250, 15)[0].tolist(),
        "sample_hash": {
            f"s{s}_it{it}_P{P}_L{L}_n{n}": sha(rng.sample_distinct(rng.stream_keys(s, it, np.arange(n)), P, L))
            for (s, it, P, L, n) in [(0, 1, 250, 15, 2000), (3, 2, 40, 7, 500), (9, 1, 125000, 28, 3000), (1, 4, 5, 5, 10), (0, 1, 17, 1, 10)]
        },
    }
    # ---- larger builds: hashes only (q=32 5k/10k/20k iteration 1)
    big = {}
    for n in (5000, 10000, 20000):
        v = pauli_view(n, 32, 0)
        lists = random_lists(v, seed=0)
        g = conflict.build(v, lists, threads=8)
        big[f"q32_n{n}"] = dict(
            n=n, q=32, seed=0, lists_sha=sha(lists.array), members_sha=sha(g.members),
            offsets_sha=sha(g.graph.offsets), neighbors_sha=sha(g.graph.neighbors),
            edge_count=int(g.edge_count), view_edges_scanned=int(g.view_edges_scanned),
            members=int(g.members.size),
        )
        print("big", n, big[f"q32_n{n}"], flush=True)
    ref["builds_hashed"] = big
    # ---- whole-run goldens (per-iteration CSR hashes of c1 + coloring hashes)
    runs = {}
    orig_build = conflict.build
    trace = []

    def tracing_build(view, lists, **kw):
        g = orig_build(view, lists, **kw)
        trace.append(dict(
            n_active=int(view.n_active), active_sha=sha(view.active), lists_sha=sha(lists.array),
            palette_base=int(lists.palette_base), palette_size=int(lists.palette_size),
            members_sha=sha(g.members), offsets_sha=sha(g.graph.offsets),
            neighbors_sha=sha(g.graph.neighbors), edge_count=int(g.edge_count),
            view_edges_scanned=int(g.view_edges_scanned),
        ))
        return g

    conflict.build = tracing_build
    try:
        specs = [("c1", 2000, 16, 0, 0, 12.5, 2.0, "dynamic")]
        specs += [(f"tout_k{k}", 120 + 60 * k, 5 + k, k, k, 12.5, 2.0, "dynamic") for k in range(5)]
        specs += [("cli_fixture", 80, 5, 1, 7, 12.5, 2.0, "dynamic")]
        specs += [(f"static_{s}", 300, 7, 2, 3, 12.5, 2.0, s) for s in ("natural", "ldf", "sdl", "random")]
        specs += [("aggressive", 400, 9, 4, 5, 3.0, 30.0, "dynamic")]
        for name, n, q, gseed, pseed, pct, alpha, strat in specs:
            trace.clear()
            v = pauli_view(n, q, gseed)
            res = pc.run(v, pc.PaletteParams(pct, alpha, seed=pseed), strategy=strat)
            runs[name] = dict(
                n=n, q=q, gen_seed=gseed, seed=pseed, palette_pct=pct, alpha=alpha, strategy=strat,
                colors=int(res.total_colors), iterations=len(res.iterations),
                peak_conflict_edges=int(res.peak_conflict_edges), oracle_edges=int(res.oracle_edges),
                color_sha=sha(res.color), colored_at_sha=sha(res.colored_at),
                records=[
                    dict(n_active=r.n_active, palette_size=r.palette_size, palette_base=r.palette_base,
                         list_size=r.list_size, conflict_vertices=r.conflict_vertices,
                         conflict_edges=r.conflict_edges, colored_unconflicted=r.colored_unconflicted,
                         colored_in_conflict=r.colored_in_conflict, uncolored=r.uncolored,
                         memory_proxy_entries=r.memory_proxy_entries, stalled=r.stalled)
                    for r in res.iterations
                ],
                builds=list(trace),
            )
            print("run", name, runs[name]["colors"], runs[name]["iterations"], flush=True)
    finally:
        conflict.build = orig_build
    ref["runs"] = runs
    # recorded by the survey run, too slow to regenerate here routinely
    ref["runs_recorded"] = {
        "q32_n50000": dict(n=50000, q=32, gen_seed=0, seed=0, palette_pct=12.5, alpha=2.0,
                           colors=7498, iterations=8, oracle_edges=624971966,
                           peak_conflict_edges=46729476, color_sha="5acbe96d9c45c44b"),
    }
    with open(os.path.join(OUT, "reference.json"), "w") as f:
        json.dump(ref, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
