"""Full-size parity at the benchmarked and north-star configurations (GPU, default suite).

Every entry of every CSR is compared, through hashes: tests/golden/scale.json holds the
iteration-1 CSR hashes of configs 2 and 3 (and 4) and whole-run colorings with per-iteration
CSR hashes, produced by the scale oracle (oracle/bucket_oracle.c, tools/make_golden_scale.py)
which tests/test_scale_oracle.py pins against the reference's own outputs — including the
reference's recorded 50k whole run.  The product side goes through the public API
(paper_2401_06713_b200.build / run -> C ABI -> sm_100a kernels) and hashes its int64 output
the same way (oracle/scale.py csr_hashes: members/offsets sha + a block hash of the
neighbors).  Reference: conflict.py:89-167, driver.py:272-385.
"""
import hashlib
import json
import os
import time

import numpy as np
import pytest

import paper_2401_06713_b200 as b200
from conftest import GOLDEN
from oracle.scale import BLOCK_ROWS, csr_hashes, sha16

pytestmark = pytest.mark.gpu

CONFIGS = {"c2": (100_000, 32), "c3": (1_000_000, 64), "c4": (4_000_000, 128),
           "q32_n50000": (50_000, 32)}


@pytest.fixture(scope="module")
def scale_gold():
    with open(os.path.join(GOLDEN, "scale.json")) as f:
        return json.load(f)


def _view(name):
    n, q = CONFIGS[name]
    return b200.pauli_view(b200.PauliSet.from_strings(b200.random_pauli_strings(n, q, seed=0)))


def _hashes(gc):
    return csr_hashes(gc.members, gc.graph.offsets, gc.graph.neighbors, gc.edge_count,
                      gc.view_edges_scanned)


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_iteration1_csr_full_hash(scale_gold, name):
    want = scale_gold["builds"][name]
    view = _view(name)
    assert sha16(view.backing.words.view(np.int64)) == want["words_sha"]
    plan = b200.plan_iteration(1, view.n_active, b200.PaletteParams(12.5, 2.0, seed=0))
    lists = b200.assign_random_lists(plan, view.active, 0)  # GPU lists at this size
    assert sha16(lists.array) == want["lists_sha"]
    t = time.perf_counter()
    gc = b200.build(view, lists)
    dt = time.perf_counter() - t
    got = _hashes(gc)
    print(f"{name}: build {dt:.3f} s, |E_c|={gc.edge_count}")
    for k in ("members_sha", "offsets_sha", "neighbors_bsha", "n_members", "edge_count",
              "view_edges_scanned"):
        assert got[k] == want[k], (k, got[k], want[k])


@pytest.mark.parametrize("name", ["q32_n50000", "c2", "c3"])
def test_whole_run_identical_coloring_full_size(scale_gold, name):
    """The whole Picasso run on the GPU: every residue build's CSR and the final coloring
    equal the oracle-driven run (q32_n50000: also the reference's own recorded run)."""
    if name not in scale_gold["runs"]:
        pytest.skip(f"no golden run for {name}")
    want = scale_gold["runs"][name]
    got = []

    def tracing(view, lists, **kw):
        gc = b200.build(view, lists, **kw)
        h = _hashes(gc)
        h.update(n_active=int(view.n_active), active_sha=sha16(view.active),
                 lists_sha=sha16(lists.array))
        got.append(h)
        return gc

    t = time.perf_counter()
    res = b200.run(_view(name), b200.PaletteParams(12.5, 2.0, seed=0), builder=tracing)
    print(f"{name}: whole run {time.perf_counter() - t:.1f} s (incl. hashing), "
          f"{res.total_colors} colors, {len(res.iterations)} iterations")
    assert len(got) == len(want["builds"])
    for it, (g, w) in enumerate(zip(got, want["builds"])):
        for k in g:
            assert g[k] == w[k], (it + 1, k, g[k], w[k])
    assert sha16(res.color) == want["color_sha"]
    assert sha16(res.colored_at) == want["colored_at_sha"]
    assert res.total_colors == want["colors"]
    assert len(res.iterations) == want["iterations"]
    assert res.oracle_edges == want["oracle_edges"]
    assert res.peak_conflict_edges == want["peak_conflict_edges"]


def test_c4_iteration1_csr_full_hash(scale_gold):
    """Config 4 (4M x 128 qubits, two-word bit planes): the whole iteration-1 CSR (7.2e9 edges)
    against the scale oracle's hashes, without the 115 GB int64 array on the host at once.
    The build is counted once over all rows (every degree, K1 over the whole triangle); the
    neighbor ids then come out through the row-range ABI (pcg_count / pcg_fill_rows) in
    chunks of whole 4096-row hash blocks, each hashed as the oracle hashes it."""
    if "c4" not in scale_gold["builds"]:
        pytest.skip("no c4 golden (tools/make_golden_scale.py --builds c4)")
    from paper_2401_06713_b200 import _native
    from paper_2401_06713_b200.conflict import stage

    want = scale_gold["builds"]["c4"]
    view = _view("c4")
    assert sha16(view.backing.words.view(np.int64)) == want["words_sha"]
    n = view.n_active
    plan = b200.plan_iteration(1, n, b200.PaletteParams(12.5, 2.0, seed=0))
    lists = b200.assign_random_lists(plan, view.active, 0)
    assert sha16(lists.array) == want["lists_sha"]
    ctx = _native.context()
    t = time.perf_counter()
    stage(view, lists, ctx)
    c = ctx.count(0, 1, 0, n)
    print(f"c4: prep + count {time.perf_counter() - t:.2f} s", flush=True)
    assert int(c.deg_sum) // 2 == want["edge_count"]
    assert int(c.pairs_in_shard - c.anticommuting) == want["view_edges_scanned"]
    deg, _ = ctx.degrees(n)
    has = deg > 0
    assert int(has.sum()) == want["n_members"]
    offsets = np.zeros(n + 1, dtype=np.int64) if has.all() else None
    assert offsets is not None, "c4 iteration 1 has a row without conflicts: compaction"
    np.cumsum(deg.astype(np.int64), out=offsets[1:])
    assert sha16(view.active[has]) == want["members_sha"]
    assert sha16(offsets) == want["offsets_sha"]
    from concurrent.futures import ThreadPoolExecutor

    digests = []
    chunk = 64 * BLOCK_ROWS
    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        for r0 in range(0, n, chunk):
            r1 = min(n, r0 + chunk)
            ctx.count(0, 1 << 22, r0, r1)  # this row range (and a negligible K1 shard)
            lo, hi = ctx.fill_rows(deg, None)
            assert (lo, hi) == (int(offsets[r0]), int(offsets[r1]))
            buf = np.empty(hi - lo, dtype=np.int64)
            ctx.fill_rows(deg, buf)
            blocks = [(b0, min(b0 + BLOCK_ROWS, r1)) for b0 in range(r0, r1, BLOCK_ROWS)]
            digests += list(ex.map(
                lambda b: hashlib.sha256(buf[offsets[b[0]] - lo:offsets[b[1]] - lo].data).digest(),
                blocks))
            del buf
    got = hashlib.sha256(b"".join(digests)).hexdigest()[:16]
    print(f"c4: full CSR hashed in {time.perf_counter() - t:.1f} s", flush=True)
    assert got == want["neighbors_bsha"]


C5 = {"c5_p20_a0.5": (20.0, 0.5), "c5_p5_a2": (5.0, 2.0), "c5_p2.5_a3": (2.5, 3.0)}


@pytest.mark.parametrize("name", sorted(C5))
def test_config5_grid_cell_full_hash(scale_gold, name):
    """Config 5 (500k x 64q, palette/alpha sweep): whole iteration-1 CSRs of grid cells from
    sparse (P' = 20%, alpha = 0.5: 7-color lists) to dense (P' = 2.5%, alpha = 3: 39-color
    lists, ~1.5k members per bucket) against the scale oracle."""
    if name not in scale_gold["builds"]:
        pytest.skip(f"no golden for {name}")
    want = scale_gold["builds"][name]
    pct, alpha = C5[name]
    view = b200.pauli_view(b200.PauliSet.from_strings(b200.random_pauli_strings(500_000, 64, seed=0)))
    plan = b200.plan_iteration(1, view.n_active, b200.PaletteParams(pct, alpha, seed=0))
    lists = b200.assign_random_lists(plan, view.active, 0)
    assert sha16(lists.array) == want["lists_sha"]
    t = time.perf_counter()
    gc = b200.build(view, lists)
    print(f"{name}: build {time.perf_counter() - t:.3f} s, |E_c|={gc.edge_count}")
    got = _hashes(gc)
    for k in ("members_sha", "offsets_sha", "neighbors_bsha", "n_members", "edge_count",
              "view_edges_scanned"):
        assert got[k] == want[k], (k, got[k], want[k])


def _check_run(res, want):
    assert sha16(res.color) == want["color_sha"]
    assert sha16(res.colored_at) == want["colored_at_sha"]
    assert res.total_colors == want["colors"]
    assert len(res.iterations) == want["iterations"]
    assert res.oracle_edges == want["oracle_edges"]
    assert res.peak_conflict_edges == want["peak_conflict_edges"]
    for r, w in zip(res.iterations, want["records"]):
        for k in ("n_active", "palette_size", "list_size", "conflict_vertices", "conflict_edges",
                  "colored_in_conflict", "uncolored"):
            assert getattr(r, k) == w[k], (r.iteration, k)


def test_whole_run_counts_only_c3_matches_the_csr_run(scale_gold):
    """driver.run(conflict_rows=False): counts-only builds (no CSR on the host) and the
    word-predicate list coloring give the c3 run of the golden (oracle CSR builds + CSR-row
    coloring), iteration by iteration."""
    want = scale_gold["runs"]["c3"]
    t = time.perf_counter()
    res = b200.run(_view("c3"), b200.PaletteParams(12.5, 2.0, seed=0), conflict_rows=False)
    print(f"c3 counts-only whole run {time.perf_counter() - t:.1f} s, {res.total_colors} colors")
    _check_run(res, want)


def test_whole_run_counts_only_c4(scale_gold):
    """Config 4 (4M x 128q, multiple Picasso iterations) as a whole run: counts-only GPU
    builds + the word-predicate coloring against the oracle's counts-only run
    (tools/make_golden_scale.py --runs-counts c4)."""
    want = scale_gold.get("runs_counts", {}).get("c4")
    if want is None:
        pytest.skip("no c4 counts-only run golden")
    t = time.perf_counter()
    res = b200.run(_view("c4"), b200.PaletteParams(12.5, 2.0, seed=0), conflict_rows=False)
    print(f"c4 counts-only whole run {time.perf_counter() - t:.1f} s, {res.total_colors} colors, "
          f"{len(res.iterations)} iterations")
    _check_run(res, want)
