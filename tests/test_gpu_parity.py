"""Parity of the CUDA builder with the reference (golden vectors) and the oracle.

Every test here calls the product path (paper_2401_06713_b200.build -> C ABI -> sm_100a
kernels).  Bit-exact equality is required everywhere: this is integer/index work.
"""

import numpy as np
import pytest

import paper_2401_06713_b200 as b200
from paper_2401_06713_b200 import _native
from paper_2401_06713_b200.conflict import last_stats, one_phase_projection
from paper_2401_06713_b200.errors import EdgeBudgetExceededError
from conftest import oracle_builder, pauli_view, random_lists, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[1, 5], ids=["k1-direct", "k1-fourrussians-8bit"])
def k1_algo(request):
    ctx = _native.context()
    ctx.option("k1_algo", request.param)
    yield request.param
    ctx.option("k1_algo", 0)


@pytest.fixture(params=[1, 2, 3], ids=["k2-gather", "k2-bucketmasks", "k2-owned"])
def k2_mode(request):
    ctx = _native.context()
    ctx.option("k2_mode", request.param)
    yield request.param
    ctx.option("k2_mode", 0)


def test_every_golden_build(golden_cases, k1_algo, k2_mode):
    for case in golden_cases:
        case.check(b200.build(case.view, case.lists))


@pytest.mark.parametrize("own_algo,own_direct,own_bitmap", [(0, 1, 1), (0, 0, 1), (0, 0, 0), (1, 0, 1)],
                         ids=["own-fourrussians-direct", "own-fourrussians-bitmap",
                              "own-fourrussians-hash", "own-perpair"])
def test_owned_mask_kernels(golden_cases, golden_ref, own_algo, own_direct, own_bitmap):
    """The owned-mask kernels (table-driven / per-pair masks; direct-mapped / bitmap /
    hashed ownership) give the reference CSR."""
    ctx = _native.context()
    ctx.option("k2_mode", 3)
    ctx.option("own_algo", own_algo)
    ctx.option("own_direct", own_direct)
    ctx.option("own_bitmap", own_bitmap)
    try:
        for case in golden_cases:
            case.check(b200.build(case.view, case.lists))
        for n in (5000, 20000):
            g = golden_ref["builds_hashed"][f"q32_n{n}"]
            v = pauli_view(n, 32, 0)
            gc = b200.build(v, random_lists(v, seed=0))
            assert (sha(gc.graph.offsets), sha(gc.graph.neighbors)) == (
                g["offsets_sha"], g["neighbors_sha"])
    finally:
        ctx.option("own_algo", 0)
        ctx.option("own_direct", 1)
        ctx.option("own_bitmap", 1)
        ctx.option("k2_mode", 0)


@pytest.mark.parametrize("fill_algo", [0, 3, 5, 6, 7],
                         ids=["auto", "lane-bitmap", "block", "segmented", "bins"])
def test_owned_fill_variants(golden_cases, fill_algo):
    ctx = _native.context()
    ctx.option("k2_mode", 3)
    ctx.option("fill_algo", fill_algo)
    try:
        for case in golden_cases:
            case.check(b200.build(case.view, case.lists))
    finally:
        ctx.option("fill_algo", 0)
        ctx.option("k2_mode", 0)


@pytest.mark.parametrize("bits,warps", [(1024, 1), (3072, 2), (12288, 2), (20480, 4),
                                        (131072, 3), (131072, 4)])
def test_segmented_fill_geometry(golden_cases, golden_ref, bits, warps):
    """Window size (1..many windows per row) and warps per block must not change a single
    entry."""
    ctx = _native.context()
    ctx.option("fill_algo", 6)
    ctx.option("seg_bits", bits)
    ctx.option("seg_warps", warps)
    try:
        for case in golden_cases:
            case.check(b200.build(case.view, case.lists))
        for n in (10000, 20000):
            g = golden_ref["builds_hashed"][f"q32_n{n}"]
            v = pauli_view(n, 32, 0)
            gc = b200.build(v, random_lists(v, seed=0))
            assert (sha(gc.graph.offsets), sha(gc.graph.neighbors)) == (
                g["offsets_sha"], g["neighbors_sha"])
    finally:
        ctx.option("fill_algo", 0)
        ctx.option("seg_bits", 0)
        ctx.option("seg_warps", 0)


@pytest.mark.parametrize("threads,groups,dcap,ecap", [
    (32, 1, 0, 0), (64, 2, 8, 32), (128, 4, 0, -1), (256, 1, 16, 0), (256, 4, 0, 64),
    (512, 16, 0, 0), (1024, 8, 24, -1), (128, 8, 0, 0), (96, 2, 0, 100)])
def test_block_fill_geometry(golden_cases, golden_ref, threads, groups, dcap, ecap):
    """Block fill: CTA size, groups per thread (1..many windows per row), descriptor chunking
    and the admitted-id list (fits / overflows into the re-decode / disabled) must not change
    a single entry."""
    ctx = _native.context()
    ctx.option("fill_algo", 5)
    ctx.option("blk_threads", threads)
    ctx.option("blk_groups", groups)
    ctx.option("blk_dcap", dcap)
    ctx.option("blk_ecap", ecap)
    try:
        for case in golden_cases:
            case.check(b200.build(case.view, case.lists))
        for n in (10000, 20000):
            g = golden_ref["builds_hashed"][f"q32_n{n}"]
            v = pauli_view(n, 32, 0)
            gc = b200.build(v, random_lists(v, seed=0))
            assert (sha(gc.graph.offsets), sha(gc.graph.neighbors)) == (
                g["offsets_sha"], g["neighbors_sha"])
    finally:
        for k in ("fill_algo", "blk_threads", "blk_groups", "blk_dcap", "blk_ecap"):
            ctx.option(k, 0)


@pytest.mark.parametrize("threads,dcap,shift", [(32, 0, 0), (128, 8, 0), (256, 0, 0), (1024, 24, 0),
                                               (128, 0, 1), (192, 0, 3), (192, 16, 5), (128, 0, -1)])
def test_bins_fill_geometry(golden_cases, golden_ref, threads, dcap, shift):
    """Bins fill (counting sort per row): CTA size, descriptor chunking and bin width must not
    change a single entry.  Wider bins (shift > 0) exercise the spill list (bins of 10-16 ids)
    and the per-row fallback (bins of more than 16 ids: list, scatter, sort from the list)."""
    ctx = _native.context()
    ctx.option("fill_algo", 7)
    ctx.option("bins_threads", threads)
    ctx.option("blk_dcap", dcap)
    ctx.option("bins_shift", shift)
    try:
        for case in golden_cases:
            case.check(b200.build(case.view, case.lists))
        for n in (10000, 20000):
            g = golden_ref["builds_hashed"][f"q32_n{n}"]
            v = pauli_view(n, 32, 0)
            gc = b200.build(v, random_lists(v, seed=0))
            assert (sha(gc.graph.offsets), sha(gc.graph.neighbors)) == (
                g["offsets_sha"], g["neighbors_sha"])
    finally:
        for k in ("fill_algo", "bins_threads", "blk_dcap", "bins_shift"):
            ctx.option(k, 0)


@pytest.mark.parametrize("n", [5000, 10000, 20000])
def test_hashed_q32_builds(golden_ref, n):
    g = golden_ref["builds_hashed"][f"q32_n{n}"]
    v = pauli_view(n, 32, 0)
    lists = random_lists(v, seed=0)
    assert sha(lists.array) == g["lists_sha"]
    gc = b200.build(v, lists)
    assert gc.edge_count == g["edge_count"]
    assert gc.view_edges_scanned == g["view_edges_scanned"]
    assert (sha(gc.members), sha(gc.graph.offsets), sha(gc.graph.neighbors)) == (
        g["members_sha"], g["offsets_sha"], g["neighbors_sha"])


@pytest.mark.parametrize("window", [4096, 8192, 32768])
def test_window_geometry_does_not_change_rows(golden_ref, window, k2_mode):
    g = golden_ref["builds_hashed"]["q32_n10000"]
    ctx = _native.context()
    ctx.option("window", window)
    try:
        v = pauli_view(10000, 32, 0)
        gc = b200.build(v, random_lists(v, seed=0))
    finally:
        ctx.option("window", 0)
    assert sha(gc.graph.neighbors) == g["neighbors_sha"]


@pytest.mark.parametrize("name", ["c1", "tout_k0", "tout_k1", "tout_k2", "tout_k3", "tout_k4",
                                  "cli_fixture", "static_natural", "static_ldf", "static_sdl",
                                  "static_random", "aggressive"])
def test_whole_run_identical_coloring(golden_ref, name):
    r = golden_ref["runs"][name]
    v = pauli_view(r["n"], r["q"], r["gen_seed"])
    res = b200.run(v, b200.PaletteParams(r["palette_pct"], r["alpha"], seed=r["seed"]),
                   strategy=r["strategy"])
    assert sha(res.color) == r["color_sha"]
    assert res.total_colors == r["colors"]
    assert len(res.iterations) == r["iterations"]
    assert res.oracle_edges == r["oracle_edges"]
    assert res.peak_conflict_edges == r["peak_conflict_edges"]


def test_per_iteration_csr_hashes_of_c1(golden_ref):
    """Every residue build of the c1 run (induced views, later palettes) hashes like the reference."""
    want = golden_ref["runs"]["c1"]["builds"]
    got = []

    def tracing(view, lists, **kw):
        gc = b200.build(view, lists, **kw)
        got.append(dict(n_active=view.n_active, active_sha=sha(view.active), lists_sha=sha(lists.array),
                        members_sha=sha(gc.members), offsets_sha=sha(gc.graph.offsets),
                        neighbors_sha=sha(gc.graph.neighbors), edge_count=gc.edge_count,
                        view_edges_scanned=gc.view_edges_scanned))
        return gc

    v = pauli_view(2000, 16, 0)
    b200.run(v, b200.PaletteParams(12.5, 2.0, seed=0), builder=tracing)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        for k in g:
            assert g[k] == w[k], k


def test_edge_budget_two_phase_and_one_phase():
    v = pauli_view(400, 6, 1)
    lists = random_lists(v, seed=3)
    full = b200.build(v, lists)
    assert b200.build(v, lists, edge_budget=full.edge_count).edge_count == full.edge_count
    with pytest.raises(EdgeBudgetExceededError) as ei:
        b200.build(v, lists, edge_budget=full.edge_count - 1)
    assert ei.value.projected == full.edge_count
    # one-phase: partial count at the first overrunning reference block
    from oracle.oracle import oracle_build

    deg_upper = oracle_build(v, lists).deg_upper
    for block_pairs, budget in ((64, 10), (4096, 500), (1 << 20, full.edge_count - 1)):
        with pytest.raises(EdgeBudgetExceededError) as ei:
            b200.build(v, lists, edge_budget=budget, two_phase=False, block_pairs=block_pairs)
        assert ei.value.projected == one_phase_projection(deg_upper, block_pairs, budget)


def test_threads_and_block_pairs_do_not_change_result():
    v = pauli_view(150, 6, 9)
    lists = random_lists(v, seed=7)
    base = b200.build(v, lists)
    for kw in (dict(threads=4), dict(block_pairs=64), dict(two_phase=False, threads=3)):
        other = b200.build(v, lists, **kw)
        assert np.array_equal(base.graph.neighbors, other.graph.neighbors)
        assert np.array_equal(base.graph.offsets, other.graph.offsets)


def test_invalid_codes_use_raw_word_predicate():
    """Hand-built words with non-Pauli 3-bit codes: the build must follow popcount(a & b)
    over the raw words exactly like the reference (pauli.py:258-268)."""
    rs = np.random.default_rng(5)
    n, q = 700, 21  # 63 bits: one word
    words = rs.integers(0, 1 << 63, size=(n, 1), dtype=np.uint64)
    ps = b200.PauliSet(["I" * q] * n, words)
    v = b200.pauli_view(ps)
    lists = random_lists(v, seed=2)
    gc = b200.build(v, lists)
    assert last_stats.raw_words_mode
    want = oracle_builder(v, lists)
    assert np.array_equal(gc.graph.neighbors, want.graph.neighbors)
    assert gc.view_edges_scanned == want.view_edges_scanned


@pytest.mark.parametrize("n", [0, 1, 2, 3])
def test_tiny_views(n):
    v = pauli_view(10, 4, 0).induce(np.arange(n))
    lists = b200.ColorLists.from_array(v.active, np.zeros((n, 1), dtype=np.int64), 0, 1)
    gc = b200.build(v, lists)
    want = oracle_builder(v, lists)
    assert np.array_equal(gc.members, want.members)
    assert np.array_equal(gc.graph.offsets, want.graph.offsets)
    assert np.array_equal(gc.graph.neighbors, want.graph.neighbors)
    assert gc.view_edges_scanned == want.view_edges_scanned
    assert gc.graph.neighbors.dtype == np.int64 and gc.graph.offsets.dtype == np.int64


@pytest.mark.parametrize("n,q", [(1500, 5), (3000, 20), (2500, 33), (5000, 64), (1200, 100),
                                 (1100, 130), (2049, 128)])
def test_commute_count_both_kernels_vs_oracle(n, q, k1_algo):
    from oracle.oracle import OracleInstance

    v = pauli_view(n, q, n + q)
    lists = random_lists(v, seed=1)
    gc = b200.build(v, lists)
    inst = OracleInstance(v.backing.words, v.active, lists)
    assert gc.view_edges_scanned == inst.commute_count()
    for i in (0, n // 3, n - 1):
        row, _ = inst.row(i)
        assert np.array_equal(gc.graph.neighbors[gc.graph.offsets[i]:gc.graph.offsets[i + 1]], row)


@pytest.mark.parametrize("n,pct", [(40000, 50.0), (60000, 45.0)])
def test_owned_direct_table_large_palette(n, pct):
    """Palettes between 14336 and 28672 colors take the 16-bit direct ownership table: the CSR
    must equal the bitmap and hash-table paths', and sampled rows the oracle's."""
    from oracle.oracle import OracleInstance

    v = pauli_view(n, 32, 5)
    lists = random_lists(v, pct=pct, seed=2)
    assert 14336 < lists.palette_size <= 28672
    ctx = _native.context()
    try:
        ctx.option("own_direct", 1)
        a = b200.build(v, lists)
        want = (sha(a.graph.offsets), sha(a.graph.neighbors), a.view_edges_scanned)
        nb, off = a.graph.neighbors.copy(), a.graph.offsets.copy()
        a = None
        ctx.option("own_direct", 0)
        b = b200.build(v, lists)  # exact color bitmap
        assert (sha(b.graph.offsets), sha(b.graph.neighbors), b.view_edges_scanned) == want
        b = None
        ctx.option("own_bitmap", 0)
        b = b200.build(v, lists)  # hash table
        assert (sha(b.graph.offsets), sha(b.graph.neighbors), b.view_edges_scanned) == want
    finally:
        ctx.option("own_direct", 1)
        ctx.option("own_bitmap", 1)
    inst = OracleInstance(v.backing.words, v.active, lists)
    for i in (0, n // 2, n - 1):
        row, _ = inst.row(i)
        assert np.array_equal(nb[off[i]:off[i + 1]], row)


@pytest.mark.parametrize("pct,alpha", [(3.0, 3.03), (0.75, 3.03)])
def test_owned_masks_shared_memory_fallbacks(pct, alpha):
    """Big buckets x long lists: the owned-mask kernel's shared memory does not fit with staged
    lists (P=600, L=30: ~1000 members) or at all (P=150, L=30: ~4000 members); the build
    drops list staging / ownership instead of failing the launch."""
    from oracle.oracle import OracleInstance

    n = 20000
    v = pauli_view(n, 32, 8)
    lists = random_lists(v, pct=pct, alpha=alpha, seed=4)
    assert lists.array.shape[1] == 30
    gc = b200.build(v, lists)
    inst = OracleInstance(v.backing.words, v.active, lists)
    assert gc.view_edges_scanned == inst.commute_count()
    nb, off = gc.graph.neighbors, gc.graph.offsets
    for i in (0, 7777, n - 1):
        row, _ = inst.row(i)
        assert np.array_equal(nb[off[i]:off[i + 1]], row)


@pytest.mark.parametrize("n,pct,alpha", [(6000, 3.0, 30.0), (20000, 3.0, 30.0)])
def test_aggressive_lists(n, pct, alpha):
    """SURVEY's aggressive corner (alpha = 30): lists of hundreds of colors (no ownership, no
    segmented fill) and, at n = 6000, lists equal to the whole palette (L = P = 180)."""
    from oracle.oracle import OracleInstance

    v = pauli_view(n, 32, 9)
    lists = random_lists(v, pct=pct, alpha=alpha, seed=6)
    L = lists.array.shape[1]
    assert L > 64
    gc = b200.build(v, lists)
    if n <= 6000:
        assert L == lists.palette_size
        want = oracle_builder(v, lists)
        assert np.array_equal(gc.graph.offsets, want.graph.offsets)
        assert np.array_equal(gc.graph.neighbors, want.graph.neighbors)
        return
    inst = OracleInstance(v.backing.words, v.active, lists)
    assert gc.view_edges_scanned == inst.commute_count()
    nb, off = gc.graph.neighbors, gc.graph.offsets
    for i in (0, n // 2, n - 1):
        row, _ = inst.row(i)
        assert np.array_equal(nb[off[i]:off[i + 1]], row)


def test_auto_bins_fill_above_block_range():
    """n > 128K ids takes the bins fill by default (and the pipelined public copy-out): the
    commuting-pair count and sampled full rows against the oracle, sortedness and offsets."""
    from oracle.oracle import OracleInstance

    n = 140_000
    v = pauli_view(n, 48, 12)
    lists = random_lists(v, seed=5)
    gc = b200.build(v, lists)
    nb, off = gc.graph.neighbors, gc.graph.offsets
    assert off[0] == 0 and off[-1] == nb.size == 2 * gc.edge_count
    inst = OracleInstance(v.backing.words, v.active, lists)
    assert gc.view_edges_scanned == inst.commute_count()
    rs = np.random.default_rng(3)
    for i in rs.choice(n, size=6, replace=False):
        row, _ = inst.row(int(i))
        assert np.array_equal(nb[off[i]:off[i + 1]], row)
        assert np.all(np.diff(row) > 0)


def test_full_size_config2_properties():
    """BASELINE config 2 (100k x 32q): the oracle cannot build it in test time, so check
    size-independent properties: commuting-pair total against the oracle's popcount sweep,
    sampled full rows against the oracle, sortedness, degree/offset consistency, symmetry of
    sampled rows."""
    from oracle.oracle import OracleInstance

    n = 100_000
    v = pauli_view(n, 32, 0)
    lists = random_lists(v, seed=0)
    gc = b200.build(v, lists)
    nb, off = gc.graph.neighbors, gc.graph.offsets
    assert off[0] == 0 and off[-1] == nb.size == 2 * gc.edge_count
    src = np.repeat(np.arange(gc.graph.n, dtype=np.int64), np.diff(off))
    same = src[1:] == src[:-1]
    assert np.all(np.diff(nb)[same] > 0)
    assert not np.any(nb == src)
    inst = OracleInstance(v.backing.words, v.active, lists)
    assert gc.view_edges_scanned == inst.commute_count()
    rs = np.random.default_rng(0)
    for i in rs.choice(n, size=12, replace=False):
        row, _ = inst.row(int(i))
        got = nb[off[i]:off[i + 1]]
        assert np.array_equal(got, row)
        for j in got[:5]:  # symmetry
            assert i in nb[off[j]:off[j + 1]]


@pytest.mark.parametrize("n,P,L,it,seed,base", [(2000, 250, 15, 1, 0, 0), (500, 40, 7, 2, 3, 100),
                                                 (3000, 125000, 28, 1, 9, 0), (10, 5, 5, 4, 1, 7),
                                                 (10, 17, 1, 1, 0, 0), (4000, 5000, 59, 3, -5, 11),
                                                 (300, 400, 394, 1, 2, 0)])
def test_gpu_palette_lists_bit_identical(n, P, L, it, seed, base):
    """csrc/rng.cu draws exactly the host splitmix64/Floyd lists (rng.py:22-70)."""
    if L > P:
        pytest.skip("L <= P")
    rs = np.random.default_rng(n)
    active = np.sort(rs.choice(10 * n, size=n, replace=False)).astype(np.int64)
    plan = b200.IterationPlan(iteration=it, palette_size=P, palette_base=base, list_size=L)
    host = b200.assign_random_lists(plan, active, seed, device=False)
    dev = b200.assign_random_lists(plan, active, seed, device=True)
    assert np.array_equal(host.array, dev.array)


def test_gpu_palette_lists_golden(golden_ref):
    plan = b200.plan_iteration(1, 2000, b200.PaletteParams(12.5, 2.0, 0))
    dev = b200.assign_random_lists(plan, np.arange(2000), 0, device=True)
    want = next(b for b in golden_ref["runs"]["c1"]["builds"] if b["n_active"] == 2000)
    assert sha(dev.array) == want["lists_sha"]


def test_whole_run_50k_recorded_golden(golden_ref):
    """The largest run the reference could finish on the survey host (50,000 x 32q, 8
    iterations, 503 s there): identical coloring (sha of the color array), color count,
    iteration count, |E| and peak |E_c|."""
    r = golden_ref["runs_recorded"]["q32_n50000"]
    v = pauli_view(r["n"], r["q"], r["gen_seed"])
    res = b200.run(v, b200.PaletteParams(r["palette_pct"], r["alpha"], seed=r["seed"]))
    assert res.total_colors == r["colors"]
    assert len(res.iterations) == r["iterations"]
    assert res.oracle_edges == r["oracle_edges"]
    assert res.peak_conflict_edges == r["peak_conflict_edges"]
    assert sha(res.color) == r["color_sha"]


def test_pinned_direct_copy_matches(golden_ref):
    """The second build reuses (and pins) the pooled host buffer: neighbor ids are copied
    straight into it and widened in place.  Both copies give the reference CSR."""
    from paper_2401_06713_b200 import hostpool

    g = golden_ref["builds_hashed"]["q32_n20000"]
    v = pauli_view(20000, 32, 0)
    lists = random_lists(v, seed=0)
    for _ in range(3):
        gc = b200.build(v, lists)
        assert gc.graph.neighbors.nbytes >= hostpool.MIN_POOLED_BYTES
        assert sha(gc.graph.neighbors) == g["neighbors_sha"]
        assert sha(gc.graph.offsets) == g["offsets_sha"]
        gc = None


def test_concurrent_builds_from_threads(golden_ref):
    """tuner.sweep(cell_workers>1) calls run() from several Python threads (tuner.py:138-141):
    each thread gets its own context and stream, the GIL is released during the native calls,
    and the pooled host buffers are never shared between live graphs."""
    import threading

    names = ["q32_n5000", "q32_n10000", "q32_n20000"]
    inputs = {}
    for nm in names:
        n = int(nm.split("_n")[1])
        v = pauli_view(n, 32, 0)
        inputs[nm] = (v, random_lists(v, seed=0))
    got, errors = {}, []

    def work(nm):
        try:
            for _ in range(2):
                gc = b200.build(*inputs[nm])
                got.setdefault(nm, []).append((sha(gc.graph.offsets), sha(gc.graph.neighbors)))
        except Exception as e:  # noqa: BLE001  (reported below)
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(nm,)) for nm in names]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for nm in names:
        g = golden_ref["builds_hashed"][nm]
        assert got[nm] == [(g["offsets_sha"], g["neighbors_sha"])] * 2


@pytest.mark.parametrize("limit", ["2", "1"])
def test_copy_out_with_a_small_openmp_team(golden_ref, limit):
    """The copy-out's decoders stride by the team OpenMP actually grants (OMP_THREAD_LIMIT
    below the requested 15-16 threads) and the pipeline's orchestrator is its own thread."""
    import os
    import subprocess
    import sys

    g = golden_ref["builds_hashed"]["q32_n20000"]
    code = (
        "import sys, hashlib, numpy as np; sys.path.insert(0, 'tests'); "
        "import paper_2401_06713_b200 as b200; from conftest import pauli_view, random_lists; "
        "v = pauli_view(20000, 32, 0); gc = b200.build(v, random_lists(v, seed=0)); "
        "h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]; "
        "print(h(gc.graph.offsets), h(gc.graph.neighbors))"
    )
    env = dict(os.environ, OMP_THREAD_LIMIT=limit)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.split()[-2:] == [g["offsets_sha"], g["neighbors_sha"]]


@pytest.mark.parametrize("n,pct,alpha", [(3000, 12.5, 2.0), (40000, 40.0, 0.6), (70000, 25.0, 1.0)])
def test_delta_copy_out_matches_widened_copy(n, pct, alpha):
    """The public build ships CSR gaps as bytes (escapes to an exception list for gaps >= 255
    and first entries) and decodes them on the host; the plain int32 copy-out (option
    d2h_mode 4) must give the same arrays, for dense and very sparse rows (long gaps) and
    for fresh (unaligned) and pooled destinations."""
    ps = b200.PauliSet.from_strings(b200.random_pauli_strings(n, 32, seed=11))
    v = b200.pauli_view(ps)
    plan = b200.plan_iteration(1, n, b200.PaletteParams(pct, alpha, seed=3))
    lists = b200.assign_random_lists(plan, v.active, 3)
    ctx = _native.context()
    try:
        ctx.option("d2h_mode", 4)
        want = b200.build(v, lists)
        ref = (want.graph.offsets.copy(), want.graph.neighbors.copy(), want.members.copy())
        want = None
        ctx.option("d2h_mode", 0)
        # (pipelined fill, pieces, chunk ids, gap width): whole-fill copy-out, default pipeline,
        # one piece, many small pieces, a piece per chunk; 16-bit and byte gaps forced
        # and the share of chunks shipped as int64 by DMA (pooled destinations are pinned)
        for pipe, pieces, chunk, gap16, dma in [(0, 0, 0, 0, 0), (1, 0, 0, 0, -1), (1, 1, 0, 1, 0),
                                                (1, 7, 4096, 2, 30), (1, 1000, 2048, 0, 50),
                                                (0, 0, 0, 1, 0), (1, 3, 0, 2, 100)]:
            ctx.option("d2h_pipe", pipe)
            ctx.option("d2h_pieces", pieces)
            ctx.option("d2h_chunk", chunk)
            ctx.option("d2h_gap16", gap16)
            ctx.option("d2h_dma", dma)
            for _ in range(2):
                got = b200.build(v, lists)
                assert np.array_equal(got.graph.offsets, ref[0])
                assert np.array_equal(got.members, ref[2])
                assert np.array_equal(got.graph.neighbors, ref[1])
                got = None
    finally:
        for k, d in (("d2h_mode", 0), ("d2h_gap16", 0), ("d2h_pipe", 1), ("d2h_pieces", 0), ("d2h_chunk", 0),
                     ("d2h_dma", -1)):
            ctx.option(k, d)


@pytest.mark.parametrize("ragged", [False, True])
def test_duplicate_colors_in_a_row(ragged):
    """A list naming one color twice (the reference ORs it into the palette mask once,
    driver.py:152-172): the device flags it in the bucket pass, the rows are deduped and the
    build matches the oracle (which builds the same set masks)."""
    n = 3000
    v = pauli_view(n, 24, 21)
    lists = random_lists(v, seed=8)
    arr = lists.array.copy()
    rs = np.random.default_rng(4)
    rows = rs.choice(n, size=40, replace=False)
    arr[rows, 1] = arr[rows, 0]  # duplicate the first color of 40 rows
    if ragged:
        rl = [arr[i, : 3 + (i % 5)].copy() for i in range(n)]
        lists = b200.ColorLists(v.active, rl, lists.palette_base, lists.palette_size)
    else:
        lists = b200.ColorLists.from_array(v.active, arr, lists.palette_base, lists.palette_size)
    gc = b200.build(v, lists)
    want = oracle_builder(v, lists)
    assert np.array_equal(gc.members, want.members)
    assert np.array_equal(gc.graph.offsets, want.graph.offsets)
    assert np.array_equal(gc.graph.neighbors, want.graph.neighbors)
    assert gc.view_edges_scanned == want.view_edges_scanned


def test_early_k1_shards_sum_to_the_whole_sweep(golden_ref):
    """The early K1 launch of a sharded build (options k1_async/k1_early/k1_shard/k1_nshards:
    the rank's shard swept beside the owned masks) is taken over by the count of the same
    shard; the shards' pairs and anticommuting counts add up to the one-shard sweep."""
    from paper_2401_06713_b200.conflict import stage

    g = golden_ref["builds_hashed"]["q32_n20000"]
    v = pauli_view(20000, 32, 0)
    lists = random_lists(v, seed=0)
    ctx = _native.context()
    n = v.n_active
    want = None
    try:
        stage(v, lists, ctx)
        c = ctx.count(0, 1, 0, n)
        want = (int(c.pairs_in_shard), int(c.anticommuting))
        for world in (2, 3):
            pairs = anti = 0
            for rank in range(world):
                for k, val in (("k1_async", 1), ("k1_early", 1), ("k1_shard", rank),
                               ("k1_nshards", world)):
                    ctx.option(k, val)
                stage(v, lists, ctx)
                c = ctx.count(rank, world, 0, n)
                pairs += int(c.pairs_in_shard)
                anti += ctx.k1_result()
            assert (pairs, anti) == want, (world, pairs, anti, want)
        assert want[0] - want[1] == g["view_edges_scanned"]
    finally:
        for k, val in (("k1_async", 0), ("k1_early", 2), ("k1_shard", 0), ("k1_nshards", 1)):
            ctx.option(k, val)
