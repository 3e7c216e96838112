"""Host-side mirror of the reference API (no GPU): encoding, RNG, plan, block geometry,
one-phase budget projection, and whole runs driven by the oracle builder."""

import math

import numpy as np
import pytest

import paper_2401_06713_b200 as b200
from paper_2401_06713_b200 import rng
from paper_2401_06713_b200.conflict import one_phase_projection
from paper_2401_06713_b200.graph import pair_chunks
from conftest import oracle_builder, pauli_view, sha


def test_encode_known_answers(golden_ref):
    enc = golden_ref["encode"]
    assert b200.random_pauli_strings(2000, 16, seed=0)[:3] == enc["c1_first3"]
    words = b200.PauliSet.from_strings(enc["c1_first3"]).words[:, 0]
    assert [f"0x{int(w):016x}" for w in words] == enc["c1_words_first3"]
    assert b200.encode("XYZI").value == enc["XYZI"] == 0b000011101110
    w22 = b200.PauliSet.from_strings(["XYZI" * 5 + "YZ"]).words.ravel()
    assert [f"0x{int(w):016x}" for w in w22] == enc["q22_words"]
    assert b200.random_pauli_strings(8, 1, seed=2, exclude_identity=True) == enc["gen_exclude_identity"]


def test_generator_hashes(golden_ref):
    import hashlib

    for key, want in golden_ref["encode"]["gen_hash"].items():
        n, rest = key.split("x")
        q, s = rest.split("s")
        text = "\n".join(b200.random_pauli_strings(int(n), int(q), seed=int(s)))
        assert hashlib.sha256(text.encode()).hexdigest()[:16] == want


def test_single_letters_and_decode():
    for ch, code in (("I", 0), ("X", 0b110), ("Y", 0b101), ("Z", 0b011)):
        assert b200.encode(ch).value == code
    s = "XYZIIZYXXZ" * 3
    assert b200.decode(b200.encode(s)) == s


def test_predicate_exhaustive_two_qubits():
    import itertools

    strings = ["".join(p) for p in itertools.product("IXYZ", repeat=2)]
    ps = b200.PauliSet.from_strings(strings)
    for a in range(16):
        for b in range(16):
            assert ps.anticommutes(a, b) == b200.anticommutes_oracle(strings[a], strings[b])


def test_bad_inputs():
    from paper_2401_06713_b200.errors import BadSymbolError, EmptyInputError, MixedLengthError

    with pytest.raises(BadSymbolError):
        b200.PauliSet.from_strings(["XQ"])
    with pytest.raises(MixedLengthError):
        b200.PauliSet.from_strings(["XX", "X"])
    with pytest.raises(EmptyInputError):
        b200.PauliSet.from_strings([])


def test_rng_known_answers(golden_ref):
    r = golden_ref["rng"]
    hexes = lambda a: [f"0x{int(x):016x}" for x in a]  # noqa: E731
    assert hexes(rng.mix64(np.array([0, 1, 2], dtype=np.uint64))) == r["mix64_0_1_2"]
    keys = rng.stream_keys(0, 1, [0, 1, 2])
    assert hexes(keys) == r["stream_keys_0_1"]
    assert hexes(rng.stream_keys(-5, 3, [0, 7, 1 << 40])) == r["stream_keys_neg"]
    assert rng.sample_distinct(keys, 250, 15)[0].tolist() == r["sample_250_15_row0"]
    import re

    for key, want in r["sample_hash"].items():
        s, it, P, L, n = map(int, re.findall(r"\d+", key))
        assert sha(rng.sample_distinct(rng.stream_keys(s, it, np.arange(n)), P, L)) == want


def test_plan_values():
    p = b200.plan_iteration(1, 1000, b200.PaletteParams(12.5, 2.0))
    assert (p.palette_size, p.list_size) == (125, round(2 * math.log(1000)))
    assert b200.plan_iteration(1, 100, b200.PaletteParams(3.0, 30.0)).list_size == 3
    esc = b200.plan_iteration(2, 1000, b200.PaletteParams(12.5, 2.0), stall_count=2)
    assert esc.palette_size == 500


def _reference_chunks(n, target):
    """graph.py:379-388 restated as the reference's loop."""
    r0 = 0
    while r0 < n - 1:
        r1, pairs = r0, 0
        while r1 < n - 1 and pairs < target:
            pairs += n - 1 - r1
            r1 += 1
        yield r0, r1
        r0 = r1


@pytest.mark.parametrize("n,target", [(2, 1), (3, 64), (150, 64), (150, 10_000), (1000, 1 << 20),
                                      (777, 1), (500, 1000)])
def test_pair_chunks_geometry(n, target):
    assert list(pair_chunks(n, target)) == list(_reference_chunks(n, target))


def test_one_phase_projection():
    rs = np.random.default_rng(3)
    deg_upper = rs.integers(0, 5, size=300)
    deg_upper[-1] = 0  # the last row has no partner j > i
    for target in (64, 1000, 1 << 20):
        for budget in (0, 10, 100, int(deg_upper.sum()) - 1):
            total = 0
            want = None
            for r0, r1 in _reference_chunks(300, target):
                total += int(deg_upper[r0:r1].sum())
                if total > budget:
                    want = total
                    break
            assert one_phase_projection(deg_upper, target, budget) == want


@pytest.mark.parametrize("name", ["c1", "tout_k0", "tout_k3", "cli_fixture", "static_sdl",
                                  "static_random", "aggressive"])
def test_whole_runs_with_oracle_builder(golden_ref, name):
    r = golden_ref["runs"][name]
    v = pauli_view(r["n"], r["q"], r["gen_seed"])
    res = b200.run(v, b200.PaletteParams(r["palette_pct"], r["alpha"], seed=r["seed"]),
                   strategy=r["strategy"], builder=oracle_builder)
    assert sha(res.color) == r["color_sha"]
    assert sha(res.colored_at) == r["colored_at_sha"]
    assert res.total_colors == r["colors"]
    assert [rec.conflict_edges for rec in res.iterations] == [x["conflict_edges"] for x in r["records"]]
    assert res.oracle_edges == r["oracle_edges"]


@pytest.mark.parametrize("seed", [0, 1, 7, 123456789])
def test_native_list_coloring_matches_python(seed):
    """pcg_color_dynamic (C++) makes the same PCG64 draws as the Python restatement."""
    from paper_2401_06713_b200 import list_coloring as lc

    for n, q, pct, alpha in ((300, 6, 12.5, 2.0), (900, 9, 3.0, 8.0), (120, 4, 30.0, 1.0)):
        v = pauli_view(n, q, seed % 1000 + n)
        plan = b200.plan_iteration(1, n, b200.PaletteParams(pct, alpha, seed))
        lists = b200.assign_random_lists(plan, v.active, seed)
        gc = oracle_builder(v, lists)
        r1 = np.random.default_rng(np.random.SeedSequence([seed, 1, 0xC01]))
        r2 = np.random.default_rng(np.random.SeedSequence([seed, 1, 0xC01]))
        r3 = np.random.default_rng(np.random.SeedSequence([seed, 1, 0xC01]))
        a = lc.color_dynamic(gc, lists, r1)  # color buckets, CSR-row adjacency
        b = lc.color_dynamic_py(gc, lists, r2)
        w = lc.color_dynamic(gc, lists, r3, view=v)  # color buckets, word-predicate adjacency
        for o in (a, w):
            assert o.colored == b.colored
            assert np.array_equal(o.uncolored, b.uncolored)
            assert o.removal_ops == b.removal_ops
        assert r1.bit_generator.state == r2.bit_generator.state == r3.bit_generator.state
        assert r1.integers(1 << 30) == r2.integers(1 << 30)


@pytest.mark.parametrize("threads,par_min", [(4, 1), (3, 16), (16, 64)])
def test_native_list_coloring_threaded_scan(threads, par_min):
    """The threaded neighbor scan (pcg_color_dynamic_mt, par_min_deg < -1) gives the color-bucket
    coloring's result (CSR-row and word adjacency), removal count and generator state, on
    graphs whose rows are far above the threshold, and both match the Python restatement."""
    from paper_2401_06713_b200 import list_coloring as lc

    for n, q, pct, alpha, seed in ((3000, 16, 12.5, 2.0, 0), (2500, 12, 4.0, 3.0, 9)):
        v = pauli_view(n, q, seed + 31)
        plan = b200.plan_iteration(1, n, b200.PaletteParams(pct, alpha, seed))
        lists = b200.assign_random_lists(plan, v.active, seed)
        gc = oracle_builder(v, lists)
        assert np.diff(gc.graph.offsets).max() > 4 * par_min
        out = []
        try:
            for thr, pm, view in ((1, -1, None), (threads, -par_min - 2, None), (1, -1, v)):
                lc.NATIVE_THREADS, lc.NATIVE_PAR_MIN_DEG = thr, pm
                r = np.random.default_rng(np.random.SeedSequence([seed, 1, 0xC01]))
                o = lc.color_dynamic(gc, lists, r, view=view)
                out.append((o.colored, list(o.uncolored), o.removal_ops, r.bit_generator.state))
        finally:
            lc.NATIVE_THREADS, lc.NATIVE_PAR_MIN_DEG = 0, -1
        assert out[0] == out[1] == out[2]
        if n <= 2500:
            r = np.random.default_rng(np.random.SeedSequence([seed, 1, 0xC01]))
            p = lc.color_dynamic_py(gc, lists, r)
            assert p.colored == out[0][0] and p.removal_ops == out[0][2]


def test_native_list_coloring_ragged_lists(golden_cases):
    from paper_2401_06713_b200 import list_coloring as lc

    case = next(c for c in golden_cases if c.meta["name"] == "ragged_lists")
    gc = oracle_builder(case.view, case.lists)
    a = lc.color_dynamic(gc, case.lists, np.random.default_rng(5))
    b = lc.color_dynamic_py(gc, case.lists, np.random.default_rng(5))
    assert a.colored == b.colored and np.array_equal(a.uncolored, b.uncolored)


def test_hostpool_never_hands_out_a_live_buffer():
    from paper_2401_06713_b200 import hostpool as hp

    hp.release()
    n = hp.MIN_POOLED_BYTES // 8 + 1000
    a = hp.empty_int64(n)
    b = hp.empty_int64(n - 10)          # a is alive -> fresh memory
    assert not np.shares_memory(a, b)
    view_of_b = b[5:]                   # keeps b's memory alive through .base
    del b
    c = hp.empty_int64(n - 20)
    assert not np.shares_memory(c, view_of_b)
    del view_of_b, a
    addr = c.__array_interface__["data"][0]
    del c
    d = hp.empty_int64(n - 30)          # the pooled buffer is free again -> reused
    assert d.__array_interface__["data"][0] == addr
    small = hp.empty_int64(10)
    assert not np.shares_memory(small, d)
    hp.release()
    assert hp.cached_bytes() == 0


def test_dedupe_rows_keeps_each_rows_distinct_colors():
    """The host side of the duplicate-color path (_native.dedupe_rows): every row keeps its
    distinct colors (ascending), uniform and ragged inputs."""
    from paper_2401_06713_b200._native import dedupe_rows

    arr = np.array([[5, 3, 5], [1, 2, 3], [7, 7, 7]], dtype=np.int64)
    d, off, L = dedupe_rows(arr.reshape(-1), None, 3, 3)
    assert L == 0 and off.tolist() == [0, 2, 5, 6]
    assert d.tolist() == [3, 5, 1, 2, 3, 7]
    d, off, _ = dedupe_rows(np.array([4, 4, 9, 1], dtype=np.int64), np.array([0, 2, 4]), 0, 2)
    assert off.tolist() == [0, 1, 3] and d.tolist() == [4, 1, 9]


def test_build_reference_and_lists_intersect_match_goldens(golden_cases):
    """The host equivalence oracle kept for API parity (conflict.py:28-39, 170-205) gives the
    reference's CSR on the small golden builds (the GPU build never calls it)."""
    from paper_2401_06713_b200.conflict import build_reference, lists_intersect

    assert lists_intersect([1, 4, 9], [2, 4]) and not lists_intersect([1, 3], [2, 4, 6])
    assert not lists_intersect([], [1])
    done = 0
    for case in golden_cases:
        if case.view.n_active > 400 or case.view.mode != "implicit-complement":
            continue
        case.check(build_reference(case.view, case.lists))
        done += 1
    assert done >= 5


def test_counts_only_run_needs_pauli_view_and_defaults():
    """driver.run(conflict_rows=False) is the default builder + coloring on a Pauli view only."""
    v = pauli_view(50, 6, 1)
    params = b200.PaletteParams(12.5, 2.0, seed=0)
    with pytest.raises(b200.errors.BadParamsError):
        b200.run(v, params, conflict_rows=False, builder=oracle_builder)
    with pytest.raises(b200.errors.BadParamsError):
        b200.run(v, params, conflict_rows=False, conflict_coloring=lambda *a, **k: None)


def test_coloring_refuses_missing_rows_without_the_view():
    """A counts-only conflict graph (rows not materialized) colors only with the Pauli view."""
    from paper_2401_06713_b200 import list_coloring as lc
    from paper_2401_06713_b200.conflict import ConflictGraph
    from paper_2401_06713_b200.graph import ExplicitGraph

    v = pauli_view(300, 6, 2)
    plan = b200.plan_iteration(1, 300, b200.PaletteParams(12.5, 2.0, 0))
    lists = b200.assign_random_lists(plan, v.active, 0)
    gc = oracle_builder(v, lists)
    bare = ConflictGraph(gc.members, ExplicitGraph(gc.graph.n, gc.graph.offsets, np.zeros(0, np.int64)),
                         gc.edge_count, gc.view_edges_scanned)
    with pytest.raises(ValueError):
        lc.color_conflict_graph(bare, lists)
    a = lc.color_conflict_graph(gc, lists)
    b = lc.color_conflict_graph(bare, lists, view=v)
    assert a.colored == b.colored and np.array_equal(a.uncolored, b.uncolored)
