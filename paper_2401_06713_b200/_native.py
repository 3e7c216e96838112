"""ctypes binding of libpicasso_b200.so (the C ABI in include/picasso_b200.h).

There is no CPU path: if the library is missing or no CUDA device is visible, every entry
point raises.  ctypes releases the GIL for the duration of each foreign call, and each host
thread gets its own ``pcg_ctx`` (contexts share nothing), so concurrent builds from several
threads (tuner.sweep with cell_workers > 1, tuner.py:138-141) are safe.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpicasso_b200.so")

PCG_OK, PCG_E_ARG, PCG_E_CUDA, PCG_E_OOM, PCG_E_COLOR, PCG_E_STATE, PCG_E_DUPLICATE = range(7)


def dedupe_rows(data: np.ndarray, off, L: int, n: int):
    """Distinct colors of every list row, as a ragged (data, offsets, 0) CSR (ascending)."""
    if off is None:
        off = np.arange(n + 1, dtype=np.int64) * L
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    order = np.lexsort((data, rows))
    d, r = data[order], rows[order]
    keep = np.ones(d.size, dtype=bool)
    keep[1:] = (d[1:] != d[:-1]) | (r[1:] != r[:-1])
    lens = np.bincount(r[keep], minlength=n)
    new_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=new_off[1:])
    return np.ascontiguousarray(d[keep], dtype=np.int64), new_off, 0


class Counts(ctypes.Structure):
    _fields_ = [
        ("n_active", ctypes.c_int64),
        ("anticommuting", ctypes.c_int64),
        ("pairs_in_shard", ctypes.c_int64),
        ("deg_sum", ctypes.c_int64),
        ("deg_upper_sum", ctypes.c_int64),
        ("members_in_range", ctypes.c_int64),
        ("raw_words_mode", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


_lib = None
_lib_lock = threading.Lock()
_VP = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32


def library():
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__; __graft_entry__.build()')")
        lib = ctypes.CDLL(LIB_PATH)
        lib.pcg_version.restype = ctypes.c_int
        lib.pcg_create.argtypes = [ctypes.c_int, ctypes.POINTER(_VP)]
        lib.pcg_destroy.argtypes = [_VP]
        lib.pcg_last_error.argtypes = [_VP]
        lib.pcg_last_error.restype = ctypes.c_char_p
        lib.pcg_set_inputs.argtypes = [_VP, _VP, _I64, _I32, _I32, _VP, _I64, _VP, _VP, _I32,
                                       _I64, _I64]
        lib.pcg_count.argtypes = [_VP, _I32, _I32, _I64, _I64, ctypes.POINTER(Counts)]
        lib.pcg_copy_degrees.argtypes = [_VP, _VP, _VP]
        lib.pcg_fill.argtypes = [_VP, _VP, _VP, _VP]
        lib.pcg_fill_rows.argtypes = [_VP, _VP, _VP, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]
        lib.pcg_count_device.argtypes = [_VP, ctypes.POINTER(Counts), ctypes.POINTER(_I32)]
        lib.pcg_fill_device.argtypes = [_VP, ctypes.POINTER(_I32)]
        lib.pcg_build_device.argtypes = [_VP, ctypes.POINTER(Counts), ctypes.POINTER(_I32)]
        lib.pcg_set_profiling.argtypes = [_VP, _I32]
        lib.pcg_kernel_times.argtypes = [_VP, _VP, _I32]
        lib.pcg_set_option.argtypes = [_VP, ctypes.c_char_p, _I64]
        lib.pcg_degrees_device.argtypes = [_VP, _VP]
        lib.pcg_prep_device.argtypes = [_VP]
        lib.pcg_fill_rows_device.argtypes = [_VP, _VP, _I32, _VP, ctypes.POINTER(_I64),
                                             ctypes.POINTER(_I64)]
        lib.pcg_assign_lists.argtypes = [_VP, _VP, _I64, ctypes.c_uint64, _I64, _I32, _I64, _VP]
        lib.pcg_assign_lists.restype = ctypes.c_int
        lib.pcg_color_dynamic.argtypes = [ctypes.c_int64, _VP, _VP, _VP, _VP, _VP, _VP, _VP]
        lib.pcg_color_dynamic.restype = ctypes.c_int
        lib.pcg_color_dynamic_mt.argtypes = [ctypes.c_int64, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                             _I32, _I64]
        lib.pcg_color_dynamic_mt.restype = ctypes.c_int
        lib.pcg_color_dynamic_words.argtypes = [ctypes.c_int64, _VP, _I32, _VP, _VP, _VP, _VP, _VP]
        lib.pcg_color_dynamic_words.restype = ctypes.c_int
        lib.pcg_validate.argtypes = [_VP, _VP, _I64, _I32, _I32, _VP, _I64, _VP, _I32, _VP,
                                     ctypes.POINTER(_I64), ctypes.POINTER(_I64)]
        lib.pcg_validate.restype = ctypes.c_int
        lib.pcg_host_register.argtypes = [_VP, ctypes.c_uint64, _I32]
        lib.pcg_host_register.restype = ctypes.c_int
        lib.pcg_k1_result.argtypes = [_VP, ctypes.POINTER(_I64)]
        lib.pcg_k1_result.restype = ctypes.c_int
        lib.pcg_last_copy_bytes.argtypes = [_VP]
        lib.pcg_last_copy_bytes.restype = ctypes.c_int64
        lib.pcg_launch_total.argtypes = [_VP]
        lib.pcg_launch_total.restype = ctypes.c_int64
        lib.pcg_stream.argtypes = [_VP]
        lib.pcg_stream.restype = _VP
        lib.pcg_exchange_buffer.argtypes = [_VP, ctypes.c_uint64, ctypes.POINTER(_VP), _VP]
        lib.pcg_exchange_buffer.restype = ctypes.c_int
        lib.pcg_exchange_map.argtypes = [_VP, _VP, ctypes.POINTER(_VP)]
        lib.pcg_exchange_map.restype = ctypes.c_int
        lib.pcg_ids_to_host.argtypes = [_VP, _VP, _I64, _VP]
        lib.pcg_ids_to_host.restype = ctypes.c_int
        for name in ("pcg_create", "pcg_destroy", "pcg_set_inputs", "pcg_count",
                     "pcg_copy_degrees", "pcg_fill", "pcg_fill_rows", "pcg_count_device",
                     "pcg_fill_device", "pcg_build_device", "pcg_set_profiling",
                     "pcg_kernel_times", "pcg_set_option", "pcg_degrees_device",
                     "pcg_fill_rows_device", "pcg_prep_device"):
            getattr(lib, name).restype = ctypes.c_int
        _lib = lib
        return lib


EXPORTED = (
    "pcg_version", "pcg_create", "pcg_destroy", "pcg_last_error", "pcg_set_inputs", "pcg_count",
    "pcg_copy_degrees", "pcg_fill", "pcg_fill_rows", "pcg_count_device", "pcg_fill_device",
    "pcg_build_device", "pcg_set_profiling", "pcg_kernel_times", "pcg_set_option", "pcg_stream",
    "pcg_degrees_device", "pcg_fill_rows_device", "pcg_prep_device", "pcg_color_dynamic",
    "pcg_assign_lists", "pcg_validate", "pcg_host_register", "pcg_last_copy_bytes",
    "pcg_k1_result", "pcg_color_dynamic_mt", "pcg_launch_total", "pcg_exchange_buffer",
    "pcg_exchange_map", "pcg_ids_to_host", "pcg_color_dynamic_words",
)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_VP)


class Context:
    """One pcg_ctx (device state of a build) bound to one CUDA device."""

    def __init__(self, device: int = 0):
        self.lib = library()
        h = _VP()
        rc = self.lib.pcg_create(int(device), ctypes.byref(h))
        if rc != PCG_OK:
            why = self.lib.pcg_last_error(None).decode(errors="replace")
            raise DeviceError(f"pcg_create(device={device}) failed with code {rc}: "
                              f"no usable CUDA device ({why})")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.pcg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, what: str):
        if rc == PCG_OK:
            return
        msg = self.lib.pcg_last_error(self.h).decode(errors="replace")
        if rc == PCG_E_COLOR:
            raise ValueError(f"{what}: {msg}")
        if rc == PCG_E_ARG:
            raise ValueError(f"{what}: {msg}")
        if rc == PCG_E_OOM:
            raise MemoryError(f"{what}: {msg}")
        raise DeviceError(f"{what} failed (code {rc}): {msg}")

    def k1_result(self) -> int:
        """Anticommuting pairs of the last count (waits for an asynchronous K1)."""
        a = _I64(0)
        self._check(self.lib.pcg_k1_result(self.h, ctypes.byref(a)), "pcg_k1_result")
        return int(a.value)

    def launch_total(self) -> int:
        return int(self.lib.pcg_launch_total(self.h))

    def last_copy_bytes(self) -> int:
        return int(self.lib.pcg_last_copy_bytes(self.h))

    def stream_handle(self) -> int:
        return int(self.lib.pcg_stream(self.h) or 0)

    def option(self, key: str, value: int):
        self._check(self.lib.pcg_set_option(self.h, key.encode(), int(value)), "pcg_set_option")

    def profiling(self, on: bool):
        self._check(self.lib.pcg_set_profiling(self.h, 1 if on else 0), "pcg_set_profiling")

    def kernel_times(self) -> list:
        out = np.zeros(5, dtype=np.float32)
        self._check(self.lib.pcg_kernel_times(self.h, _ptr(out), 5), "pcg_kernel_times")
        return out.tolist()

    def set_inputs(self, words: np.ndarray, num_qubits: int, active: np.ndarray,
                   list_data: np.ndarray, list_off: np.ndarray | None, list_len: int,
                   palette_base: int, palette_size: int):
        for attempt in range(2):
            self._keep = (words, active, list_data, list_off)
            rc = self.lib.pcg_set_inputs(
                self.h, _ptr(words), int(words.shape[0]), int(words.shape[1]), int(num_qubits),
                _ptr(active), int(active.size), _ptr(list_data), _ptr(list_off), int(list_len),
                int(palette_base), int(palette_size))
            if rc != PCG_E_DUPLICATE or attempt:
                break
            # a row names a color twice: the reference's palette mask is a set (driver.py:
            # 152-172, conflict.py:72-78 ANDs mask rows), so the build sees each row's distinct
            # colors.  The device flags it during the bucket pass; the rows are deduped here
            # once and staged again (never happens for lists drawn by assign_random_lists).
            list_data, list_off, list_len = dedupe_rows(list_data, list_off, list_len,
                                                        int(active.size))
        self._check(rc, "pcg_set_inputs")

    def count(self, shard: int = 0, nshards: int = 1, row_begin: int = 0,
              row_end: int | None = None, n: int | None = None) -> Counts:
        c = Counts()
        if row_end is None:
            row_end = n
        self._check(self.lib.pcg_count(self.h, shard, nshards, row_begin, row_end, ctypes.byref(c)),
                    "pcg_count")
        return c

    def degrees(self, rows: int) -> tuple:
        deg = np.zeros(rows, dtype=np.int32)
        degu = np.zeros(rows, dtype=np.int32)
        self._check(self.lib.pcg_copy_degrees(self.h, _ptr(deg), _ptr(degu)), "pcg_copy_degrees")
        return deg, degu

    def fill(self, members: np.ndarray, offsets: np.ndarray, neighbors: np.ndarray):
        self._check(self.lib.pcg_fill(self.h, _ptr(members), _ptr(offsets), _ptr(neighbors)),
                    "pcg_fill")

    def fill_rows(self, global_deg: np.ndarray, neighbors: np.ndarray | None) -> tuple:
        lo, hi = _I64(0), _I64(0)
        g = np.ascontiguousarray(global_deg, dtype=np.int32)
        self._check(self.lib.pcg_fill_rows(self.h, _ptr(g), _ptr(neighbors), ctypes.byref(lo),
                                           ctypes.byref(hi)), "pcg_fill_rows")
        return int(lo.value), int(hi.value)

    def prep_device(self):
        self._check(self.lib.pcg_prep_device(self.h), "pcg_prep_device")

    def degrees_device(self, deg_ptr: int):
        self._check(self.lib.pcg_degrees_device(self.h, _VP(deg_ptr)), "pcg_degrees_device")

    def fill_rows_device(self, gdeg_ptr: int, maxdeg: int, out_ptr: int | None) -> tuple:
        lo, hi = _I64(0), _I64(0)
        self._check(self.lib.pcg_fill_rows_device(self.h, _VP(gdeg_ptr), int(maxdeg),
                                                  _VP(out_ptr) if out_ptr else None,
                                                  ctypes.byref(lo), ctypes.byref(hi)),
                    "pcg_fill_rows_device")
        return int(lo.value), int(hi.value)

    def exchange_buffer(self, nbytes: int) -> tuple:
        """(device pointer, 64-byte IPC handle) of this context's exported exchange buffer."""
        p, h = _VP(), ctypes.create_string_buffer(64)
        self._check(self.lib.pcg_exchange_buffer(self.h, ctypes.c_uint64(max(int(nbytes), 16)),
                                                 ctypes.byref(p), h), "pcg_exchange_buffer")
        return int(p.value), bytes(h.raw)

    def exchange_map(self, handle: bytes) -> int:
        """A peer's exchange buffer mapped into this device's address space (cached)."""
        p = _VP()
        hb = ctypes.create_string_buffer(bytes(handle), 64)
        self._check(self.lib.pcg_exchange_map(self.h, hb, ctypes.byref(p)), "pcg_exchange_map")
        return int(p.value)

    def ids_to_host(self, src_ptr: int, out: np.ndarray) -> None:
        """int32 ids at a device pointer -> the int64 host array ``out`` (widened)."""
        assert out.dtype == np.int64 and out.flags.c_contiguous
        self._check(self.lib.pcg_ids_to_host(self.h, _VP(src_ptr), int(out.size), _ptr(out)),
                    "pcg_ids_to_host")

    def assign_lists(self, active: np.ndarray, base_key: int, P: int, L: int, base: int) -> np.ndarray:
        active = np.ascontiguousarray(active, dtype=np.int64)
        out = np.empty((active.size, L), dtype=np.int64)
        self._check(self.lib.pcg_assign_lists(self.h, _ptr(active), int(active.size),
                                              ctypes.c_uint64(base_key), int(P), int(L), int(base),
                                              _ptr(out)), "pcg_assign_lists")
        return out

    def validate(self, words: np.ndarray, num_qubits: int, active: np.ndarray,
                 color: np.ndarray, cap: int) -> tuple:
        """Exhaustive properness check on the device: (violations, edges, first pairs)."""
        words = np.ascontiguousarray(words, dtype=np.uint64)
        active = np.ascontiguousarray(active, dtype=np.int64)
        color = np.ascontiguousarray(color, dtype=np.int64)
        pairs = np.empty((max(int(cap), 1), 2), dtype=np.int64)
        nv, ne = _I64(0), _I64(0)
        self._check(self.lib.pcg_validate(self.h, _ptr(words), int(words.shape[0]),
                                          int(words.shape[1]), int(num_qubits), _ptr(active),
                                          int(active.size), _ptr(color), int(cap), _ptr(pairs),
                                          ctypes.byref(nv), ctypes.byref(ne)), "pcg_validate")
        return int(nv.value), int(ne.value), pairs[:min(int(cap), int(nv.value))]

    def count_device(self) -> tuple:
        c = Counts()
        n = _I32(0)
        self._check(self.lib.pcg_count_device(self.h, ctypes.byref(c), ctypes.byref(n)),
                    "pcg_count_device")
        return c, int(n.value)

    def build_device(self) -> tuple:
        c = Counts()
        n = _I32(0)
        self._check(self.lib.pcg_build_device(self.h, ctypes.byref(c), ctypes.byref(n)),
                    "pcg_build_device")
        return c, int(n.value)

    def fill_device(self) -> int:
        n = _I32(0)
        self._check(self.lib.pcg_fill_device(self.h, ctypes.byref(n)), "pcg_fill_device")
        return int(n.value)


def host_register(a: np.ndarray, on: bool = True) -> bool:
    """Pin/unpin a numpy buffer for direct DMA (cudaHostRegister); False if it failed."""
    return library().pcg_host_register(_ptr(a), ctypes.c_uint64(a.nbytes), 1 if on else 0) == PCG_OK


_tls = threading.local()


def context(device: int | None = None) -> Context:
    """The calling thread's context on ``device`` (default: $PICASSO_DEVICE or LOCAL_RANK or 0)."""
    if device is None:
        device = int(os.environ.get("PICASSO_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    cache = getattr(_tls, "ctxs", None)
    if cache is None:
        cache = _tls.ctxs = {}
    ctx = cache.get(device)
    if ctx is None:
        ctx = cache[device] = Context(device)
    return ctx
