"""The scale oracle (oracle/bucket_oracle.c, bucket intersection, O(|E_c|) memory) pinned
against the reference's own outputs and against the dense-mask oracle.

It is the checker for configs 2-4 (tests/golden/scale.json, tools/make_golden_scale.py), so
it must agree with the reference everywhere the reference itself could be run.
"""

import numpy as np
import pytest

import paper_2401_06713_b200 as b200
from conftest import pauli_view, random_lists, sha
from oracle.oracle import oracle_build
from oracle.scale import ScaleOracle, csr_hashes, neighbors_block_sha, scale_build


def _same(a, b):
    assert np.array_equal(a.members, b.members)
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.neighbors, b.neighbors)
    assert a.edge_count == b.edge_count
    assert a.view_edges_scanned == b.view_edges_scanned


def test_scale_oracle_matches_every_golden_build(golden_cases):
    """All 23 reference builds (ragged lists, duplicates, word-boundary qubit counts, induced
    subsets, n = 2 ...), bit-exact."""
    for case in golden_cases:
        case.check(scale_build(case.view, case.lists, threads=3))


@pytest.mark.parametrize("n", [5000, 10000, 20000])
def test_scale_oracle_matches_hashed_q32_builds(golden_ref, n):
    g = golden_ref["builds_hashed"][f"q32_n{n}"]
    v = pauli_view(n, 32, 0)
    lists = random_lists(v, seed=0)
    o = scale_build(v, lists)
    assert (sha(o.members), sha(o.offsets), sha(o.neighbors)) == (
        g["members_sha"], g["offsets_sha"], g["neighbors_sha"])
    assert o.edge_count == g["edge_count"]
    assert o.view_edges_scanned == g["view_edges_scanned"]


def test_scale_oracle_c1_run_per_iteration_hashes(golden_ref):
    """The whole c1 run driven by the scale oracle: every residue build and the coloring equal
    the reference's."""
    from paper_2401_06713_b200.conflict import ConflictGraph
    from paper_2401_06713_b200.graph import ExplicitGraph

    want = golden_ref["runs"]["c1"]
    got = []

    def builder(view, lists, **kw):
        o = scale_build(view, lists)
        got.append(dict(members_sha=sha(o.members), offsets_sha=sha(o.offsets),
                        neighbors_sha=sha(o.neighbors), edge_count=o.edge_count,
                        view_edges_scanned=o.view_edges_scanned))
        return ConflictGraph(o.members, ExplicitGraph(int(o.members.size), o.offsets, o.neighbors),
                             o.edge_count, o.view_edges_scanned)

    res = b200.run(pauli_view(2000, 16, 0), b200.PaletteParams(12.5, 2.0, seed=0), builder=builder)
    assert sha(res.color) == want["color_sha"] and res.total_colors == want["colors"]
    assert len(got) == len(want["builds"])
    for g, w in zip(got, want["builds"]):
        for k in g:
            assert g[k] == w[k], k


@pytest.mark.parametrize("seed", range(6))
def test_scale_oracle_matches_dense_oracle_random(seed):
    """Random cases the goldens do not cover: ragged lists with duplicated colors, palettes
    not a multiple of 64, colors in the mask's padding range, invalid 3-bit codes."""
    from paper_2401_06713_b200.driver import ColorLists
    from paper_2401_06713_b200.graph import EdgeOracleView

    rs = np.random.default_rng(100 + seed)
    n = int(rs.integers(2, 900))
    q = int(rs.choice([3, 21, 22, 40, 64, 100]))
    nw = (3 * q + 63) // 64
    if seed % 2:
        words = rs.integers(0, 1 << 62, size=(n + 5, nw), dtype=np.uint64)  # any 3-bit codes
    else:
        words = b200.PauliSet.from_strings(b200.random_pauli_strings(n + 5, q, seed=seed)).words
    ps = b200.PauliSet(["I" * q] * (n + 5), np.ascontiguousarray(words, dtype=np.uint64))
    active = np.sort(rs.choice(n + 5, n, replace=False)).astype(np.int64)
    view = EdgeOracleView(ps, "implicit-complement", active=active)
    P = int(rs.integers(1, 300))
    base = int(rs.integers(0, 50))
    span = 64 * ((P + 63) // 64)  # the mask's legal range (driver.py:152-172)
    rows = [base + rs.integers(0, span, size=int(rs.integers(1, 12))) for _ in range(n)]
    lists = ColorLists(active, rows, base, P)
    _same(scale_build(view, lists, threads=4), oracle_build(view, lists, threads=4))


def test_scale_oracle_block_hash_matches_full_arrays():
    v = pauli_view(3000, 20, 2)
    lists = random_lists(v, seed=2)
    full = scale_build(v, lists)
    want = csr_hashes(full.members, full.offsets, full.neighbors, full.edge_count,
                      full.view_edges_scanned)
    for block in (1, 7, 4096):
        assert neighbors_block_sha(full.offsets, full.neighbors, block) == (
            want["neighbors_bsha"] if block == 4096 else
            neighbors_block_sha(full.offsets, full.neighbors, block))
    o = ScaleOracle(v.backing.words, v.active, lists, threads=3, chunk_rows=97)
    assert o.hashes() == want
    o.close()


def test_scale_oracle_rejects_colors_outside_the_mask():
    from paper_2401_06713_b200.driver import ColorLists

    v = pauli_view(10, 4, 0)
    lists = ColorLists(v.active, [np.array([70])] * 10, 0, 5)  # 64*ceil(5/64) = 64 <= 70
    with pytest.raises(ValueError):
        ScaleOracle(v.backing.words, v.active, lists)


def test_scale_oracle_thread_and_chunk_independent():
    v = pauli_view(2500, 12, 3)
    lists = random_lists(v, seed=1)
    a = ScaleOracle(v.backing.words, v.active, lists, threads=1, chunk_rows=4096).build()
    b = ScaleOracle(v.backing.words, v.active, lists, threads=6, chunk_rows=31).build()
    _same(a, b)
    assert np.array_equal(a.deg_upper, b.deg_upper)
