"""ORACLE — test infrastructure only.

ctypes front end for ``liboracle.so`` (``conflict_oracle.c``), the plain-C restatement of
the reference conflict-graph builder (``/root/reference/pkg/src/palettecolor/conflict.py:89-167``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` and
``--impl reference`` legs) may import this module, and only as the checker or the timed
CPU baseline.  Nothing under ``paper_2401_06713_b200/`` imports it.

Pinned against the golden vectors in ``tests/golden`` (``tests/test_oracle.py``), which
``tools/make_golden.py`` produced by running the reference package itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_ptr = ctypes.c_void_p


def build_library() -> str:
    """Compile liboracle.so in place (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    srcs = ("conflict_oracle.c", "bucket_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(os.path.join(_HERE, s)) for s in srcs
    ):
        build_library()
    lib = ctypes.CDLL(_LIB_PATH)
    lib.oracle_make_masks.argtypes = [_ptr, _ptr, _i64, _i64, _i64, _ptr]
    lib.oracle_make_masks.restype = ctypes.c_int
    lib.oracle_mask_words.argtypes = [_i64]
    lib.oracle_mask_words.restype = _i64
    lib.oracle_build_count.argtypes = [_ptr, _i64, _ptr, _i64, _ptr, _i64, ctypes.c_int, _ptr, _ptr]
    lib.oracle_build_fill.argtypes = [_ptr, _i64, _ptr, _i64, _ptr, _i64, ctypes.c_int, _ptr, _ptr]
    lib.oracle_commute_count.argtypes = [_ptr, _i64, _ptr, _i64, ctypes.c_int]
    lib.oracle_commute_count.restype = _i64
    lib.oracle_csr_assemble.argtypes = [_i64, _ptr, _ptr, _ptr, _ptr, _ptr]
    lib.oracle_csr_assemble.restype = _i64
    lib.oracle_row.argtypes = [_ptr, _i64, _ptr, _i64, _ptr, _i64, _i64, _ptr, _ptr]
    lib.oracle_row.restype = _i64
    lib.oracle_scan_rows.argtypes = [_ptr, _i64, _ptr, _i64, _ptr, _i64, _i64, _i64, _ptr, _ptr]
    lib.oracle_scan_rows.restype = _i64
    _lib = lib
    return lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class OracleCSR:
    members: np.ndarray
    offsets: np.ndarray
    neighbors: np.ndarray
    edge_count: int
    view_edges_scanned: int
    deg_upper: np.ndarray  # admitted j>i per local row (for the one-phase budget projection)


def _list_csr(lists) -> tuple[np.ndarray, np.ndarray]:
    """Colors of each active row as CSR (handles ColorLists.array and ragged .rows)."""
    arr = getattr(lists, "array", None)
    if arr is not None:
        arr = np.ascontiguousarray(arr, dtype=np.int64)
        n, L = arr.shape
        return arr.reshape(-1), np.arange(0, (n + 1) * L, L, dtype=np.int64)
    rows = [np.asarray(r, dtype=np.int64) for r in lists.rows]
    off = np.zeros(len(rows) + 1, dtype=np.int64)
    off[1:] = np.cumsum([r.size for r in rows])
    data = np.concatenate(rows) if rows else np.zeros(0, dtype=np.int64)
    return np.ascontiguousarray(data), off


class OracleInstance:
    """Inputs of one build, prepared the way the reference prepares them."""

    def __init__(self, words: np.ndarray, active: np.ndarray, lists, threads: int = 0):
        self.lib = _load()
        self.words = np.ascontiguousarray(words, dtype=np.uint64)
        self.nwords = int(self.words.shape[1])
        self.active = np.ascontiguousarray(active, dtype=np.int64)
        self.n = int(self.active.size)
        self.threads = threads or (os.cpu_count() or 1)
        data, off = _list_csr(lists)
        self.mwords = int(self.lib.oracle_mask_words(int(lists.palette_size)))
        self.masks = np.zeros((max(self.n, 1), self.mwords), dtype=np.uint64)
        rc = self.lib.oracle_make_masks(
            _p(data), _p(off), self.n, int(lists.palette_base), int(lists.palette_size), _p(self.masks)
        )
        if rc != 0:
            raise ValueError("color outside the palette")

    def commute_count(self) -> int:
        return int(
            self.lib.oracle_commute_count(
                _p(self.words), self.nwords, _p(self.active), self.n, self.threads
            )
        )

    def build(self) -> OracleCSR:
        n = self.n
        deg_upper = np.zeros(max(n, 1), dtype=np.int64)
        seen_upper = np.zeros(max(n, 1), dtype=np.int64)
        self.lib.oracle_build_count(
            _p(self.words), self.nwords, _p(self.active), n, _p(self.masks), self.mwords,
            self.threads, _p(deg_upper), _p(seen_upper),
        )
        deg_upper = deg_upper[:n]
        row_pos = np.zeros(n + 1, dtype=np.int64)
        row_pos[1:] = np.cumsum(deg_upper)
        total = int(row_pos[-1])
        v_arr = np.zeros(max(total, 1), dtype=np.int64)
        self.lib.oracle_build_fill(
            _p(self.words), self.nwords, _p(self.active), n, _p(self.masks), self.mwords,
            self.threads, _p(row_pos), _p(v_arr),
        )
        members_local = np.zeros(max(n, 1), dtype=np.int64)
        offsets = np.zeros(n + 2, dtype=np.int64)
        neighbors = np.zeros(max(2 * total, 1), dtype=np.int64)
        nm = int(
            self.lib.oracle_csr_assemble(
                n, _p(row_pos), _p(v_arr), _p(members_local), _p(offsets), _p(neighbors)
            )
        )
        return OracleCSR(
            members=self.active[members_local[:nm]],
            offsets=offsets[: nm + 1].copy(),
            neighbors=neighbors[: 2 * total].copy(),
            edge_count=total,
            view_edges_scanned=int(seen_upper[:n].sum()),
            deg_upper=deg_upper.copy(),
        )

    def row(self, i: int) -> tuple[np.ndarray, int]:
        """Full conflict row of local vertex i (ascending local ids) and its commuting count."""
        out = np.zeros(max(self.n, 1), dtype=np.int64)
        seen = np.zeros(1, dtype=np.int64)
        k = int(
            self.lib.oracle_row(
                _p(self.words), self.nwords, _p(self.active), self.n, _p(self.masks),
                self.mwords, int(i), _p(out), _p(seen),
            )
        )
        return out[:k].copy(), int(seen[0])

    def scan_rows(self, lo: int, hi: int) -> tuple[int, int, int]:
        """(pairs, commuting, admitted) for upper-triangle rows [lo, hi) — CPU baseline work."""
        pairs = np.zeros(1, dtype=np.int64)
        seen = np.zeros(1, dtype=np.int64)
        adm = int(
            self.lib.oracle_scan_rows(
                _p(self.words), self.nwords, _p(self.active), self.n, _p(self.masks),
                self.mwords, int(lo), int(hi), _p(pairs), _p(seen),
            )
        )
        return int(pairs[0]), int(seen[0]), adm


def oracle_build(view, lists, threads: int = 0) -> OracleCSR:
    """Oracle CSR for an implicit-complement view (duck-typed: .active, .backing.words)."""
    return OracleInstance(view.backing.words, view.active, lists, threads).build()
