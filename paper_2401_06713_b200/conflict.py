"""Conflict-graph construction on the B200 — the drop-in for palettecolor.conflict.build.

``build(view, lists, *, edge_budget=None, threads=1, block_pairs=1<<20, two_phase=True)``
has the reference's signature, inputs, outputs and errors
(/root/reference/pkg/src/palettecolor/conflict.py:89-167):

  * inputs   view.active (sorted original ids), view.backing.words (packed Pauli words),
             lists.array / lists.rows aligned with view.active, lists.palette_base/size;
  * output   ConflictGraph(members, ExplicitGraph(n_c, offsets, neighbors), edge_count,
             view_edges_scanned) — int64 arrays, canonical CSR (members ascending, rows
             strictly ascending compact ids), bit-identical to the reference;
  * errors   EdgeBudgetExceededError(projected, budget) before any output is allocated —
             the caller's own class when the view comes from the reference package
             (_error_types), so the reference's handlers and tests catch it.
             Two-phase: projected = exact total (conflict.py:117-118).  One-phase: the
             cumulative count at the first reference pair block whose running total exceeds
             the budget (conflict.py:138-142), reproduced from per-row upper degrees.

All work runs on the GPU through the C ABI (count pass -> budget check -> fill pass).
``threads`` and ``block_pairs`` only shaped the reference's CPU scan; the result never
depended on them (test_conflict.py:112-121), so they are accepted and ignored.  There is no
CPU fallback: a missing library or device raises.

If the caller passes the reference's own objects, the result is built from the reference's
own ConflictGraph/ExplicitGraph classes, so isinstance checks keep working.
"""

from __future__ import annotations

import importlib
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native, hostpool
from .errors import DeviceError, EdgeBudgetExceededError
from .graph import ExplicitGraph, pair_chunks

__all__ = ["ConflictGraph", "lists_intersect", "build", "build_counts", "build_reference",
           "BuildStats"]


@dataclass
class ConflictGraph:
    """Per-iteration conflict graph: ``graph`` vertex k is original vertex ``members[k]``."""

    members: np.ndarray
    graph: ExplicitGraph
    edge_count: int
    view_edges_scanned: int

    def original_edges(self) -> tuple:
        src = np.repeat(np.arange(self.graph.n, dtype=np.int64), self.graph.degrees())
        keep = src < self.graph.neighbors
        return self.members[src[keep]], self.members[self.graph.neighbors[keep]]

    def to_edge_list_text(self) -> str:
        u, v = self.original_edges()
        lines = [f"{a} {b}" for a, b in zip(u, v)]
        return "\n".join(lines) + ("\n" if lines else "")


@dataclass
class BuildStats:
    """Side information of the last build on this thread (for benchmarks and tests)."""

    n_active: int = 0
    raw_words_mode: bool = False
    deg_upper_sum: int = 0


last_stats = BuildStats()


def lists_intersect(a, b) -> bool:
    """Sorted-list intersection test (conflict.py:28-39)."""
    i = j = 0
    while i < len(a) and j < len(b):
        if a[i] == b[j]:
            return True
        if a[i] < b[j]:
            i += 1
        else:
            j += 1
    return False


def _caller_package(view):
    mod = type(view).__module__
    pkg = mod.rsplit(".", 1)[0] if "." in mod else mod
    return pkg if pkg and pkg != __package__ else None


def _result_types(view):
    """ConflictGraph / ExplicitGraph classes of the caller's package (duck-typed drop-in)."""
    pkg = _caller_package(view)
    if pkg:
        try:
            cg = importlib.import_module(pkg + ".conflict").ConflictGraph
            eg = importlib.import_module(pkg + ".graph").ExplicitGraph
            return cg, eg
        except (ImportError, AttributeError):
            pass
    return ConflictGraph, ExplicitGraph


_device_error_types: dict = {}


def _error_types(view):
    """(EdgeBudgetExceededError, DeviceError) to raise for this caller.

    A caller of the reference package (palettecolor views, e.g. after ``install_into``)
    gets the reference's own EdgeBudgetExceededError (errors.py:76-84), so its
    ``except EdgeBudgetExceededError`` (cli.py:446, exit code 4) and its tests'
    ``pytest.raises`` (test_conflict.py:93-98) catch it; and a DeviceError that also derives
    from the reference's PaletteColorError root, so ``except PaletteColorError`` sees device
    failures too.  Callers of this package get this package's classes.
    """
    pkg = _caller_package(view)
    if pkg:
        try:
            errs = importlib.import_module(pkg + ".errors")
            budget = errs.EdgeBudgetExceededError
            root = errs.PaletteColorError
        except (ImportError, AttributeError):
            return EdgeBudgetExceededError, DeviceError
        dev = _device_error_types.get(root)
        if dev is None:
            dev = type("DeviceError", (DeviceError, root), {"__module__": __name__})
            _device_error_types[root] = dev
        return budget, dev
    return EdgeBudgetExceededError, DeviceError


def _lists_as_csr(lists, n: int):
    """(data int64, offsets int64 or None, L) with rows aligned to view.active."""
    arr = getattr(lists, "array", None)
    if arr is not None:
        arr = np.ascontiguousarray(arr, dtype=np.int64)
        if arr.ndim != 2 or arr.shape[0] != n:
            raise ValueError(f"color lists have {arr.shape[0]} rows, view has {n} active vertices")
        return arr.reshape(-1), None, int(arr.shape[1])
    rows = [np.asarray(r, dtype=np.int64) for r in lists.rows]
    if len(rows) != n:
        raise ValueError(f"color lists have {len(rows)} rows, view has {n} active vertices")
    lens = np.fromiter((r.size for r in rows), dtype=np.int64, count=n)
    if n and lens.min() == lens.max():
        return np.ascontiguousarray(np.concatenate(rows)), None, int(lens[0])
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    data = np.concatenate(rows) if n else np.zeros(0, dtype=np.int64)
    return np.ascontiguousarray(data), off, 0


def one_phase_projection(deg_upper: np.ndarray, block_pairs: int, budget: int) -> int:
    """Running admitted count at the first reference block that exceeds ``budget``
    (conflict.py:131-142 over graph.py:379-388 blocks)."""
    n = int(deg_upper.size)
    cum = np.concatenate([[0], np.cumsum(deg_upper.astype(np.int64))])
    for r0, r1 in pair_chunks(n, block_pairs):
        if cum[r1] > budget:
            return int(cum[r1])
    return int(cum[-1])


def stage(view, lists, ctx: Optional[_native.Context] = None) -> _native.Context:
    """Copy one build's inputs to the device (K0 runs there); returns the context."""
    if view.mode != "implicit-complement":
        raise NotImplementedError(
            "the B200 builder implements the Pauli (implicit-complement) oracle; explicit "
            f"graph views ({view.mode!r}) are outside its scope")
    ctx = ctx or _native.context()
    words = np.ascontiguousarray(view.backing.words, dtype=np.uint64)
    active = np.ascontiguousarray(view.active, dtype=np.int64)
    n = int(active.size)
    data, off, L = _lists_as_csr(lists, n)
    ctx.set_inputs(words, int(view.backing.num_qubits), active, data, off, L,
                   int(lists.palette_base), int(lists.palette_size))
    return ctx


def build(view, lists, *, edge_budget: Optional[int] = None, threads: int = 1,
          block_pairs: int = 1 << 20, two_phase: bool = True):
    """Scan all active pairs on the GPU and return the canonical conflict CSR."""
    budget_error, device_error = _error_types(view)
    try:
        return _build(view, lists, edge_budget, block_pairs, two_phase, budget_error)
    except DeviceError as e:
        if isinstance(e, device_error):
            raise
        raise device_error(*e.args) from e


def _build(view, lists, edge_budget, block_pairs, two_phase, budget_error):
    CG, EG = _result_types(view)
    ctx = _native.context()
    n = view.n_active
    # the commuting-pair sweep (view_edges_scanned only) runs on a side stream, launched by
    # the input prep as soon as the bit planes exist, next to the bucket prep, the
    # conflict-row passes and the copy-out; its count is collected after the fill
    ctx.option("k1_async", 1)
    try:
        stage(view, lists, ctx)
        c = ctx.count(0, 1, 0, n)
    finally:
        ctx.option("k1_async", 0)
    total = int(c.deg_sum) // 2
    last_stats.n_active = n
    last_stats.raw_words_mode = bool(c.raw_words_mode)
    last_stats.deg_upper_sum = int(c.deg_upper_sum)
    if edge_budget is not None and total > edge_budget:
        if two_phase:
            raise budget_error(total, edge_budget)
        _, degu = ctx.degrees(n)
        raise budget_error(one_phase_projection(degu, block_pairs, edge_budget), edge_budget)
    nm = int(c.members_in_range)
    members = np.empty(nm, dtype=np.int64)
    offsets = np.empty(nm + 1, dtype=np.int64)
    neighbors = hostpool.empty_int64(2 * total)
    ctx.fill(members, offsets, neighbors)
    scanned = int(c.pairs_in_shard - ctx.k1_result())
    if nm == 0:
        offsets[0] = 0
    return CG(members=members, graph=EG(n=nm, offsets=offsets, neighbors=neighbors),
              edge_count=total, view_edges_scanned=scanned)


def build_counts(view, lists, *, edge_budget: Optional[int] = None, threads: int = 1,
                 block_pairs: int = 1 << 20, two_phase: bool = True):
    """The build's counts without its rows: members, CSR offsets, edge_count and
    view_edges_scanned of ``build`` (same kernels up to the count pass: K0, K1, owned masks,
    K2c), with ``graph.neighbors`` left empty (not materialized).

    For consumers that need only the conflict vertices — the list coloring with the Pauli
    view tests adjacency inside color buckets on the words (list_coloring.color_dynamic) —
    so that a run at config 4 does not move a 115 GB CSR per iteration.  Same errors as
    ``build``.
    """
    budget_error, device_error = _error_types(view)
    CG, EG = _result_types(view)
    try:
        ctx = _native.context()
        n = view.n_active
        ctx.option("k1_async", 0)
        stage(view, lists, ctx)
        c = ctx.count(0, 1, 0, n)
        total = int(c.deg_sum) // 2
        if edge_budget is not None and total > edge_budget:
            if two_phase:
                raise budget_error(total, edge_budget)
            _, degu = ctx.degrees(n)
            raise budget_error(one_phase_projection(degu, block_pairs, edge_budget), edge_budget)
        deg, _ = ctx.degrees(n)
    except DeviceError as e:
        if isinstance(e, device_error):
            raise
        raise device_error(*e.args) from e
    has = deg > 0
    members = np.ascontiguousarray(np.asarray(view.active, dtype=np.int64)[has])
    offsets = np.zeros(members.size + 1, dtype=np.int64)
    np.cumsum(deg[has].astype(np.int64), out=offsets[1:])
    return CG(members=members, graph=EG(n=int(members.size), offsets=offsets,
                                        neighbors=np.zeros(0, dtype=np.int64)),
              edge_count=total, view_edges_scanned=int(c.pairs_in_shard - c.anticommuting))


def build_reference(view, lists):
    """The reference's naive O(n^2 L) equivalence oracle (conflict.py:170-205), host Python.

    Public API parity only — ``build`` never calls it.
    """
    active = view.active
    n = active.size
    rows = [lists.colors_for(int(v)) for v in active]
    us, vs, seen = [], [], 0
    for a in range(n):
        for b in range(a + 1, n):
            if view.has_edge(int(active[a]), int(active[b])):
                seen += 1
                if lists_intersect(rows[a], rows[b]):
                    us.append(a)
                    vs.append(b)
    u = np.array(us, dtype=np.int64)
    v = np.array(vs, dtype=np.int64)
    touched = np.union1d(u, v)
    members = active[touched] if touched.size else np.zeros(0, dtype=np.int64)
    if touched.size:
        g = ExplicitGraph.from_edges(int(touched.size), np.searchsorted(touched, u),
                                     np.searchsorted(touched, v))
    else:
        g = ExplicitGraph(n=0, offsets=np.zeros(1, dtype=np.int64), neighbors=np.zeros(0, dtype=np.int64))
    return ConflictGraph(members=members, graph=g, edge_count=int(u.size), view_edges_scanned=seen)
