"""ORACLE — test infrastructure only (scale oracle).

ctypes front end for the bucket-intersection restatement of the reference conflict build
(``bucket_oracle.c``; ``/root/reference/pkg/src/palettecolor/conflict.py:89-167``) and the
CSR hash the full-size GPU parity tests compare against.

Only ``tests/``, ``tools/make_golden_scale.py`` and ``bench.py``'s CPU legs may import this
module, and only as the checker.  Nothing under ``paper_2401_06713_b200/`` imports it.

Hash of a canonical CSR (``csr_hashes``): ``members_sha`` / ``offsets_sha`` = first 16 hex
digits of sha256 over the int64 little-endian array (the ``sha`` used by the golden files);
``neighbors_bsha`` = sha256 over the concatenated sha256 digests of the int64 neighbor ids of
consecutive blocks of ``BLOCK_ROWS`` compact rows (a checksum of checksums: the blocks hash
in parallel on either side, and nothing needs the whole neighbor array at once).
"""

from __future__ import annotations

import ctypes
import hashlib
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from .oracle import _list_csr, _load, _p

BLOCK_ROWS = 4096
_i64 = ctypes.c_int64
_ptr = ctypes.c_void_p


def _lib():
    lib = _load()
    if not getattr(lib, "_bk_ready", False):
        lib.bk_open.argtypes = [_ptr, _i64, _ptr, _i64, _ptr, _ptr, _i64, _i64]
        lib.bk_open.restype = _ptr
        lib.bk_close.argtypes = [_ptr]
        lib.bk_set_compact.argtypes = [_ptr, _ptr]
        lib.bk_degrees.argtypes = [_ptr, _i64, _i64, _ptr, _ptr]
        lib.bk_degrees.restype = ctypes.c_int
        lib.bk_emit.argtypes = [_ptr, _i64, _i64, _ptr]
        lib.bk_emit.restype = _i64
        lib.bk_commute_count.argtypes = [_ptr, _i64, _i64, ctypes.c_int]
        lib.bk_commute_count.restype = _i64
        lib._bk_ready = True
    return lib


def sha16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).data).hexdigest()[:16]


def _block_ranges(nm: int, block_rows: int):
    return [(k, min(k + block_rows, nm)) for k in range(0, nm, block_rows)]


def neighbors_block_sha(offsets: np.ndarray, neighbors: np.ndarray, block_rows: int = BLOCK_ROWS,
                        threads: int = 0) -> str:
    """Block hash of an int64 neighbor array (see module docstring), in parallel threads."""
    nm = int(offsets.size) - 1
    offsets = np.asarray(offsets)
    if neighbors.dtype != np.int64:
        raise TypeError("neighbors must be int64")

    def one(r):
        lo, hi = int(offsets[r[0]]), int(offsets[r[1]])
        return hashlib.sha256(np.ascontiguousarray(neighbors[lo:hi]).data).digest()

    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        digests = list(ex.map(one, _block_ranges(nm, block_rows)))
    return hashlib.sha256(b"".join(digests)).hexdigest()[:16]


def csr_hashes(members, offsets, neighbors, edge_count, view_edges_scanned) -> dict:
    return {"members_sha": sha16(members), "offsets_sha": sha16(offsets),
            "neighbors_bsha": neighbors_block_sha(np.asarray(offsets), np.asarray(neighbors)),
            "n_members": int(np.asarray(members).size), "edge_count": int(edge_count),
            "view_edges_scanned": int(view_edges_scanned)}


@dataclass
class ScaleCSR:
    members: np.ndarray
    offsets: np.ndarray
    neighbors: np.ndarray
    edge_count: int
    view_edges_scanned: int
    deg_upper: np.ndarray


class ScaleOracle:
    """One build's inputs in color buckets (bucket_oracle.c bk_open)."""

    def __init__(self, words, active, lists, threads: int = 0, chunk_rows: int = 2048):
        self.lib = _lib()
        self.words = np.ascontiguousarray(words, dtype=np.uint64)
        self.active = np.ascontiguousarray(active, dtype=np.int64)
        self.n = int(self.active.size)
        self.threads = threads or (os.cpu_count() or 1)
        self.chunk = chunk_rows
        self._data, self._off = _list_csr(lists)
        if self._off.size != self.n + 1:
            raise ValueError("color lists are not aligned with the active set")
        self.h = self.lib.bk_open(_p(self.words), int(self.words.shape[1]), _p(self.active), self.n,
                                  _p(self._data), _p(self._off), int(lists.palette_base),
                                  int(lists.palette_size))
        if not self.h:
            raise ValueError("color outside the palette mask range (or out of memory)")
        self._cid = None

    def close(self):
        if self.h:
            self.lib.bk_close(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _ranges(self, lo=0, hi=None):
        hi = self.n if hi is None else hi
        return [(k, min(k + self.chunk, hi)) for k in range(lo, hi, self.chunk)]

    def degrees(self, upper: bool = False):
        deg = np.zeros(max(self.n, 1), dtype=np.int64)
        degu = np.zeros(max(self.n, 1), dtype=np.int64) if upper else None

        def one(r):
            rc = self.lib.bk_degrees(self.h, r[0], r[1], _p(deg[r[0]:]),
                                     _p(degu[r[0]:]) if upper else None)
            if rc:
                raise MemoryError("bk_degrees")

        with ThreadPoolExecutor(self.threads) as ex:
            list(ex.map(one, self._ranges()))
        return deg[:self.n], (degu[:self.n] if upper else None)

    def commute_count(self) -> int:
        return int(self.lib.bk_commute_count(self.h, 0, self.n, self.threads))

    def _compaction(self, deg):
        keep = deg > 0
        members_local = np.flatnonzero(keep).astype(np.int64)
        cid = np.full(max(self.n, 1), -1, dtype=np.int64)
        cid[members_local] = np.arange(members_local.size, dtype=np.int64)
        self._cid = cid
        self.lib.bk_set_compact(self.h, _p(cid))
        offsets = np.zeros(members_local.size + 1, dtype=np.int64)
        np.cumsum(deg[members_local], out=offsets[1:])
        return members_local, offsets

    def build(self, scanned: bool = True) -> ScaleCSR:
        """The full canonical CSR (int64), like conflict.build's output."""
        deg, degu = self.degrees(upper=True)
        members_local, offsets = self._compaction(deg)
        nb = np.empty(int(offsets[-1]), dtype=np.int64)
        starts = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(deg, out=starts[1:])

        def one(r):
            w = self.lib.bk_emit(self.h, r[0], r[1], _p(nb[starts[r[0]]:]) if nb.size else None)
            if w != starts[r[1]] - starts[r[0]]:
                raise RuntimeError("bk_emit wrote an unexpected row length")

        with ThreadPoolExecutor(self.threads) as ex:
            list(ex.map(one, self._ranges()))
        return ScaleCSR(members=self.active[members_local], offsets=offsets, neighbors=nb,
                        edge_count=int(deg.sum()) // 2,
                        view_edges_scanned=self.commute_count() if scanned else -1,
                        deg_upper=degu)

    def hashes(self, scanned: bool = True, block_rows: int = BLOCK_ROWS) -> dict:
        """csr_hashes() of the build without holding the whole neighbor array."""
        deg, _ = self.degrees()
        members_local, offsets = self._compaction(deg)
        nm = int(members_local.size)

        def one(r):
            k0, k1 = r
            lo, hi = int(offsets[k0]), int(offsets[k1])
            buf = np.empty(max(hi - lo, 1), dtype=np.int64)
            # compact rows k0..k1 are local rows members_local[k0..k1]; rows in between have
            # no partners, so emitting the local span writes exactly these rows
            w = self.lib.bk_emit(self.h, int(members_local[k0]), int(members_local[k1 - 1]) + 1,
                                 _p(buf))
            if w != hi - lo:
                raise RuntimeError("bk_emit wrote an unexpected block length")
            return hashlib.sha256(buf[:hi - lo].data).digest()

        with ThreadPoolExecutor(self.threads) as ex:
            digests = list(ex.map(one, _block_ranges(nm, block_rows)))
        return {"members_sha": sha16(self.active[members_local]), "offsets_sha": sha16(offsets),
                "neighbors_bsha": hashlib.sha256(b"".join(digests)).hexdigest()[:16],
                "n_members": nm, "edge_count": int(deg.sum()) // 2,
                "view_edges_scanned": self.commute_count() if scanned else -1}


def scale_build(view, lists, threads: int = 0) -> ScaleCSR:
    o = ScaleOracle(view.backing.words, view.active, lists, threads)
    try:
        return o.build()
    finally:
        o.close()
