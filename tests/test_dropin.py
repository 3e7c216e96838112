"""The drop-in boundary against the real reference package (CPU; this container only).

``install_into(palettecolor)`` must route the reference's own ``conflict.build`` (and, through
it, ``driver.run``, driver.py:21,313) to this package for Pauli views, return the reference's
own result classes, and raise the reference's own exception classes (errors.py:76-84), so the
reference's handlers (cli.py:441-454) and tests (test_conflict.py:88-99) keep working.

No GPU here: the device is stood in for by a fake context backed by the scale oracle
(test infrastructure), so the host half of ``build`` — staging, budget logic, result types,
error mapping — runs unchanged.  Without the stand-in, the product must fail loudly.
"""

import os
import sys

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")


@pytest.fixture(scope="module")
def pc():
    sys.path.insert(0, REF_SRC)
    try:
        import palettecolor
    finally:
        sys.path.remove(REF_SRC)
    yield palettecolor


@pytest.fixture
def installed(pc):
    import paper_2401_06713_b200 as b200

    orig_conflict, orig_pkg = pc.conflict.build, pc.build
    b200.install_into(pc)
    yield pc
    pc.conflict.build = orig_conflict
    pc.build = orig_pkg
    if hasattr(pc.conflict, "_reference_build"):
        del pc.conflict._reference_build


class FakeCounts:
    pass


class OracleDevice:
    """Stands in for _native.Context: the same methods, answered by the scale oracle."""

    def __init__(self, fail_count=False):
        self.fail_count = fail_count

    def option(self, key, value):
        pass

    def set_inputs(self, words, num_qubits, active, data, off, L, base, P):
        from oracle.scale import ScaleOracle

        class _L:
            pass

        lists = _L()
        n = active.size
        if off is None:
            lists.array = data.reshape(n, L) if n else np.zeros((0, max(L, 1)), np.int64)
        else:
            lists.array = None
            lists.rows = [data[off[k]:off[k + 1]] for k in range(n)]
        lists.palette_base, lists.palette_size = base, P
        self.active = active
        self.o = ScaleOracle(words, active, lists, threads=2)
        self.full = self.o.build()

    def count(self, shard, nshards, r0, r1):
        from paper_2401_06713_b200.errors import DeviceError

        if self.fail_count:
            raise DeviceError("pcg_count failed (code 7): simulated launch failure")
        c = FakeCounts()
        n = self.active.size
        c.deg_sum = 2 * self.full.edge_count
        c.raw_words_mode = 0
        c.deg_upper_sum = self.full.edge_count
        c.members_in_range = self.full.members.size
        c.pairs_in_shard = n * (n - 1) // 2
        return c

    def degrees(self, n):
        d = np.diff(self.full.offsets)
        deg = np.zeros(n, np.int32)
        deg[np.searchsorted(self.active, self.full.members)] = d
        return deg, self.full.deg_upper.astype(np.int32)

    def fill(self, members, offsets, neighbors):
        members[:] = self.full.members
        offsets[:] = self.full.offsets
        neighbors[:] = self.full.neighbors

    def k1_result(self):
        n = self.active.size
        return n * (n - 1) // 2 - self.full.view_edges_scanned


@pytest.fixture
def oracle_device(monkeypatch):
    from paper_2401_06713_b200 import _native

    dev = OracleDevice()
    monkeypatch.setattr(_native, "context", lambda device=None: dev)
    return dev


def _ref_inputs(pc, n=300, q=8, seed=1):
    view = pc.pauli_view(pc.PauliSet.from_strings(pc.random_pauli_strings(n, q, seed=seed)))
    plan = pc.plan_iteration(1, n, pc.PaletteParams(12.5, 2.0, seed=seed))
    lists = pc.assign_random_lists(plan, view.active, seed)
    return view, lists


def test_install_routes_pauli_views_and_returns_reference_types(installed, oracle_device):
    pc = installed
    view, lists = _ref_inputs(pc)
    got = pc.conflict.build(view, lists)
    want = pc.conflict._reference_build(view, lists)
    assert type(got) is pc.conflict.ConflictGraph
    assert type(got.graph) is pc.graph.ExplicitGraph
    assert np.array_equal(got.members, want.members)
    assert np.array_equal(got.graph.offsets, want.graph.offsets)
    assert np.array_equal(got.graph.neighbors, want.graph.neighbors)
    assert (got.edge_count, got.view_edges_scanned) == (want.edge_count, want.view_edges_scanned)
    assert pc.build is pc.conflict.build


@pytest.mark.parametrize("two_phase,block_pairs", [(True, 1 << 20), (False, 64), (False, 4096)])
def test_budget_error_is_the_reference_class(installed, oracle_device, two_phase, block_pairs):
    """test_conflict.py:88-99 and cli.py:446 catch palettecolor.errors.EdgeBudgetExceededError."""
    pc = installed
    view, lists = _ref_inputs(pc)
    full = pc.conflict._reference_build(view, lists)
    budget = full.edge_count // 3
    with pytest.raises(pc.errors.EdgeBudgetExceededError) as got:
        pc.conflict.build(view, lists, edge_budget=budget, two_phase=two_phase,
                          block_pairs=block_pairs)
    with pytest.raises(pc.errors.EdgeBudgetExceededError) as want:
        pc.conflict._reference_build(view, lists, edge_budget=budget, two_phase=two_phase,
                                     block_pairs=block_pairs)
    assert (got.value.projected, got.value.budget) == (want.value.projected, want.value.budget)
    assert isinstance(got.value, pc.errors.PaletteColorError)


def test_device_error_is_a_reference_error(installed, monkeypatch):
    pc = installed
    from paper_2401_06713_b200 import _native
    from paper_2401_06713_b200.errors import DeviceError

    dev = OracleDevice(fail_count=True)
    monkeypatch.setattr(_native, "context", lambda device=None: dev)
    view, lists = _ref_inputs(pc, n=40)
    with pytest.raises(pc.errors.PaletteColorError) as e:
        pc.conflict.build(view, lists)
    assert isinstance(e.value, DeviceError) and isinstance(e.value, RuntimeError)


def test_no_device_fails_loudly(installed):
    """No CUDA device here: the product raises (a reference-catchable error), never falls
    back to a CPU path."""
    pc = installed
    view, lists = _ref_inputs(pc, n=40)
    with pytest.raises(pc.errors.PaletteColorError):
        pc.conflict.build(view, lists)


def test_explicit_views_keep_the_reference_builder(installed):
    pc = installed
    g = pc.gnp_graph(60, 0.3, seed=2)
    view = pc.graph_view(g)
    plan = pc.plan_iteration(1, 60, pc.PaletteParams(12.5, 2.0, seed=2))
    lists = pc.assign_random_lists(plan, view.active, 2)
    got = pc.conflict.build(view, lists)  # no device needed: the reference builder runs
    want = pc.conflict._reference_build(view, lists)
    assert np.array_equal(got.graph.neighbors, want.graph.neighbors)


def test_reference_driver_run_through_the_dropin(installed, oracle_device, pc):
    """palettecolor.run (driver.py:272-385, unchanged) calls the installed build for every
    residue iteration; the coloring equals the reference's own run."""
    import paper_2401_06713_b200 as b200

    view = pc.pauli_view(pc.PauliSet.from_strings(pc.random_pauli_strings(250, 7, seed=3)))
    params = pc.PaletteParams(12.5, 2.0, seed=3)
    calls = []
    routed = pc.conflict.build

    def spy(v, lists, **kw):
        calls.append(v.n_active)
        return routed(v, lists, **kw)

    pc.conflict.build = spy
    try:
        got = pc.run(view, params)
    finally:
        pc.conflict.build = routed
    pc.conflict.build = pc.conflict._reference_build
    try:
        want = pc.run(view, params)
    finally:
        pc.conflict.build = routed
    assert len(calls) == len(want.iterations) > 1
    assert np.array_equal(got.color, want.color)
    assert got.total_colors == want.total_colors
    assert b200.conflict.last_stats.n_active == calls[-1]
