"""ctypes binding of libtidq.so (the C ABI declared in include/tidq.h).

This is the only place the package touches native code.  The library is built
in-tree (``paper_1807_01409_b200/libtidq.so``) by ``__graft_entry__.build()`` /
``python -m paper_1807_01409_b200.build``.  There is no CPU fallback: if the
library or a CUDA device is missing, :func:`lib` / :func:`context` raise.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref
from ctypes import (
    POINTER,
    Structure,
    c_char_p,
    c_int,
    c_int32,
    c_int64,
    c_uint8,
    c_uint32,
    c_uint64,
    c_void_p,
)

import numpy as np

from . import errors

LIB_NAME = "libtidq.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

# ---- constants mirrored from include/tidq.h ---------------------------------
OK = 0
E_INVALID = -1
E_CUDA = -2
E_NOMEM = -3
E_TOO_MANY_KEYS = -4
E_ROW_CAP = -5
E_NCCL = -6
E_UNSUPPORTED = -7
E_IO = -8
E_BAD_MAGIC = -9
E_BAD_VERSION = -10
E_TRUNCATED = -11
E_PARSE = -12

MAX_KEYS = 32
MAX_STREAMS = 32
MAX_OUT = 4
MAX_FILTERS = 2

OUT_S, OUT_P, OUT_O, OUT_INDEX, OUT_MARKS, OUT_ANSWER, OUT_LOCAL = range(7)
EQ_SP, EQ_SO, EQ_PO = 1, 2, 4
U32, I64, U8 = 0, 1, 2
DTYPES = {U32: np.dtype(np.uint32), I64: np.dtype(np.int64), U8: np.dtype(np.uint8)}


class SynthParams(Structure):
    _fields_ = [
        ("n_triples", c_uint64),
        ("base_index", c_uint64),
        ("seed", c_uint64),
        ("n_p", c_uint32),
        ("n_e", c_uint32),
    ]


class StreamSpec(Structure):
    _fields_ = [
        ("select", c_uint32),
        ("eq_flags", c_uint32),
        ("n_out", c_int32),
        ("out", c_int32 * MAX_OUT),
        ("answer_key", c_int32),
        ("n_filters", c_int32),
        ("filter_slot", c_int32 * MAX_FILTERS),
        ("filter", c_void_p * MAX_FILTERS),
        ("capacity_hint", c_uint64),
        ("key_bitmap", c_void_p),
        ("key_bitmap_slot", c_int32),
    ]


class ScanSpec(Structure):
    _fields_ = [
        ("n_keys", c_int32),
        ("keys", (c_uint32 * 3) * MAX_KEYS),
        ("n_streams", c_int32),
        ("streams", StreamSpec * MAX_STREAMS),
        ("flags", c_uint32),
        ("write_counts", c_void_p),
    ]


SCAN_ASYNC = 1  # tidq.h TIDQ_SCAN_ASYNC
SCAN_CONCAT = 2  # tidq.h TIDQ_SCAN_CONCAT


_P = c_void_p  # opaque handles
_PP = POINTER(c_void_p)

_SIGNATURES = {
    "tidq_abi_version": ([], c_int),
    "tidq_last_error": ([], c_char_p),
    "tidq_device_count": ([POINTER(c_int)], c_int),
    "tidq_ctx_create": ([c_int, _PP], c_int),
    "tidq_ctx_destroy": ([_P], c_int),
    "tidq_ctx_sync": ([_P], c_int),
    "tidq_ctx_launches": ([_P, POINTER(c_uint64)], c_int),
    "tidq_host_alloc": ([c_uint64, _PP], c_int),
    "tidq_host_free": ([_P], c_int),
    "tidq_timer_begin": ([_P], c_int),
    "tidq_timer_end": ([_P, POINTER(ctypes.c_double)], c_int),
    "tidq_profile_enable": ([_P, c_int], c_int),
    "tidq_profile_read": ([_P, c_char_p, POINTER(ctypes.c_double), POINTER(c_uint64), POINTER(c_uint64)], c_int),
    "tidq_profile_reset": ([_P], c_int),
    "tidq_store_upload": ([_P, _P, c_uint64, c_uint64, _PP], c_int),
    "tidq_store_generate": ([_P, POINTER(SynthParams), _P, _PP], c_int),
    "tidq_store_load_tid": ([_P, c_char_p, c_uint64, _PP], c_int),
    "tidq_store_load_tid_range": ([_P, c_char_p, c_uint64, c_uint64, c_uint64, _PP], c_int),
    "tidq_ctx_mem_info": ([_P, POINTER(c_uint64), POINTER(c_uint64)], c_int),
    "tidq_store_gather_cols": ([_P, _P, c_int32, c_int32, _P, _PP], c_int),
    "tidq_store_gather_cols_multi": ([_P, _P, c_int32, _P, _P, _PP], c_int),
    "tidq_tables_semijoin": ([c_int32, _P, _P, c_uint64, _P], c_int),
    "tidq_store_info": ([_P, POINTER(c_uint64), POINTER(c_uint64)], c_int),
    "tidq_store_download": ([_P, c_uint64, c_uint64, _P], c_int),
    "tidq_store_gather": ([_P, _P, c_uint64, _P], c_int),
    "tidq_store_col_max": ([_P, c_int32, POINTER(c_uint32)], c_int),
    "tidq_store_pred_hist": ([_P, c_uint32, _P], c_int),
    "tidq_store_free": ([_P], c_int),
    "tidq_scan": ([_P, POINTER(ScanSpec), _PP], c_int),
    "tidq_scan_host": ([_P, _P, c_uint64, c_uint64, POINTER(ScanSpec), _PP], c_int),
    "tidq_table_info": ([_P, POINTER(c_uint64), POINTER(c_int32)], c_int),
    "tidq_table_ncols": ([_P, POINTER(c_int32)], c_int),
    "tidq_table_col_dtype": ([_P, c_int32, POINTER(c_int32)], c_int),
    "tidq_table_download_col": ([_P, c_int32, _P], c_int),
    "tidq_table_upload_u32": ([_P, c_int32, _P, c_uint64, _PP], c_int),
    "tidq_table_free": ([_P], c_int),
    "tidq_table_concat": ([_P, c_int32, _P, c_int32, _P, _PP], c_int),
    "tidq_table_project": ([_P, c_int32, _P, _PP], c_int),
    "tidq_table_filter_bitmap": ([_P, c_int32, _P, _PP], c_int),
    "tidq_table_unique_col": ([_P, c_int32, _PP], c_int),
    "tidq_distinct": ([_P, c_int32, _P, _PP], c_int),
    "tidq_distinct_bound": ([_P, c_int32, _P, c_uint64, _PP], c_int),
    "tidq_join": ([_P, c_int32, _P, c_int32, c_int32, _P, c_int32, _P, c_int64, c_int32, c_uint64, _P, _P, _PP,
                   POINTER(c_uint64)], c_int),
    "tidq_merge_join_pairs": ([_P, _P, c_uint64, _P, c_uint64, _PP], c_int),
    "tidq_argsort_u32": ([_P, _P, c_uint64, _P, _P], c_int),
    "tidq_store_pcodes": ([_P, _P, ctypes.c_uint32], c_int),
    "tidq_store_so": ([_P, c_int32], c_int),
    "tidq_ctx_trim": ([_P], c_int),
    "tidq_debug_radix_sort": ([_P, c_int32, _P, _P, c_uint64, c_int32, c_int32, POINTER(ctypes.c_double)], c_int),
    "tidq_comm_unique_id": ([_P], c_int),
    "tidq_comm_create": ([_P, _P, c_int32, c_int32, _PP], c_int),
    "tidq_comm_destroy": ([_P], c_int),
    "tidq_comm_stats": ([_P, c_int32, POINTER(c_uint64), POINTER(ctypes.c_double)], c_int),
    "tidq_table_partition": ([_P, c_int32, _P, c_int32, _PP, _P], c_int),
    "tidq_table_alltoallv": ([_P, _P, _P, _PP, _P], c_int),
    "tidq_table_allgather": ([_P, _P, _PP], c_int),
    "tidq_comm_allreduce_u64": ([_P, _P, _P, c_int32], c_int),
    "tidq_bitmap_upload": ([_P, _P, c_uint64, _PP], c_int),
    "tidq_bitmap_create": ([_P, c_uint64, _PP], c_int),
    "tidq_bitmap_free": ([_P], c_int),
    "tidq_convert_nt": ([c_char_p, c_char_p, c_int, c_int, _P, POINTER(c_void_p)], c_int),
    "tidq_convert_free": ([c_void_p], c_int),
}

class ConvertReport(Structure):
    """tidq_convert_report (include/tidq.h)."""

    _fields_ = [("triples", c_uint64), ("terms", c_uint64), ("distinct", c_uint64 * 3),
                ("skipped_lines", c_uint64), ("parse_errors", c_uint64), ("file_bytes", c_uint64 * 4),
                ("first_error_line", c_uint64), ("first_error_offset", c_uint64),
                ("io_errno", c_int32), ("io_path", ctypes.c_char * 4096)]


_lib = None
_lib_lock = threading.Lock()


def exported_symbols() -> list[str]:
    """Every entry point the binding expects libtidq.so to export."""
    return list(_SIGNATURES)


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libtidq.so and declare every prototype (no GPU needed)."""
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_1807_01409_b200.build` "
            "(there is no CPU fallback)"
        )
    cdll = ctypes.CDLL(path)
    for name, (argtypes, restype) in _SIGNATURES.items():
        fn = getattr(cdll, name)
        fn.argtypes = argtypes
        fn.restype = restype
    return cdll


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                _lib = load()
    return _lib


def check(rc: int) -> None:
    """Map a libtidq status code to the reference's exception classes."""
    if rc == OK:
        return
    msg = lib().tidq_last_error().decode("utf-8", "replace")
    if rc == E_TOO_MANY_KEYS:
        raise errors.TooManySubqueries(msg)
    if rc == E_ROW_CAP:
        raise errors.ResourceLimit(msg)
    if rc == E_INVALID:
        raise ValueError(msg)
    if rc == E_NOMEM:
        raise MemoryError(msg)
    if rc == E_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == E_IO:
        raise OSError(msg)
    if rc == E_BAD_MAGIC:
        raise errors.BadMagic(msg)
    if rc == E_BAD_VERSION:
        raise errors.BadVersion(msg)
    if rc == E_TRUNCATED:
        raise errors.TruncatedFile(msg)
    if rc == E_PARSE:
        raise errors.ParseError.from_message(msg)
    raise RuntimeError(f"libtidq error {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


# ---- pinned host memory for result downloads --------------------------------


class PinnedPool:
    """Page-locked host blocks for downloaded result columns.

    A D2H copy into fresh pageable numpy memory runs at ~4 GB/s on the GPU
    box (page faults + the driver's bounce buffer); into page-locked memory
    it runs at the PCIe rate (~55 GB/s).  Columns of at least MIN_BYTES are
    therefore returned as ordinary numpy arrays whose buffer is a pooled
    pinned block; the block goes back to the pool when the array (and every
    view of it) is garbage-collected.  Blocks are power-of-two sized; the
    pool keeps at most CACHE_BYTES of idle blocks.
    """

    MIN_BYTES = 1 << 20
    CACHE_BYTES = 4 << 30

    def __init__(self):
        self._free: dict[int, list[int]] = {}
        self._idle = 0
        self._lock = threading.Lock()

    @staticmethod
    def _size_class(nbytes: int) -> int:
        return 1 << max(20, (nbytes - 1).bit_length())

    def _take(self, size: int) -> int:
        with self._lock:
            lst = self._free.get(size)
            if lst:
                self._idle -= size
                return lst.pop()
        p = c_void_p()
        call("tidq_host_alloc", size, ctypes.byref(p))
        return p.value

    def _give(self, addr: int, size: int) -> None:
        with self._lock:
            if self._idle + size <= self.CACHE_BYTES:
                self._free.setdefault(size, []).append(addr)
                self._idle += size
                return
        try:
            lib().tidq_host_free(c_void_p(addr))
        except Exception:
            pass

    def empty(self, n: int, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        nbytes = n * dtype.itemsize
        if nbytes < self.MIN_BYTES:
            return np.empty(n, dtype=dtype)
        size = self._size_class(nbytes)
        addr = self._take(size)
        buf = (ctypes.c_uint8 * nbytes).from_address(addr)
        weakref.finalize(buf, self._give, addr, size)
        return np.frombuffer(buf, dtype=dtype, count=n)


_pinned_pool = PinnedPool()


def pinned_empty(n: int, dtype) -> np.ndarray:
    """np.empty(n, dtype), page-locked (pooled) when large enough."""
    return _pinned_pool.empty(n, dtype)


# ---- device contexts ---------------------------------------------------------


class Context:
    """One CUDA device: stream, memory pool, scan scratch (tidq_ctx)."""

    def __init__(self, device: int = 0):
        self.device = device
        h = c_void_p()
        call("tidq_ctx_create", device, ctypes.byref(h))
        self.handle = h

    def sync(self) -> None:
        call("tidq_ctx_sync", self.handle)

    def trim(self) -> None:
        """Return unused pooled device memory to the driver (tidq_ctx_trim)."""
        call("tidq_ctx_trim", self.handle)

    def mem_info(self) -> tuple[int, int]:
        """(free, total) device bytes."""
        f, t = c_uint64(), c_uint64()
        call("tidq_ctx_mem_info", self.handle, ctypes.byref(f), ctypes.byref(t))
        return f.value, t.value

    def timer_begin(self) -> None:
        call("tidq_timer_begin", self.handle)

    def timer_end(self) -> float:
        """Milliseconds on the ctx stream since timer_begin (CUDA events)."""
        ms = ctypes.c_double()
        call("tidq_timer_end", self.handle, ctypes.byref(ms))
        return ms.value

    def profile(self, on: bool = True) -> None:
        call("tidq_profile_enable", self.handle, int(on))

    def profile_reset(self) -> None:
        call("tidq_profile_reset", self.handle)

    def profile_read(self, kernel: str) -> tuple[float, int, int]:
        """(total ms, launches, algorithmic bytes) of a profiled hot kernel."""
        ms = ctypes.c_double()
        n = c_uint64()
        b = c_uint64()
        call("tidq_profile_read", self.handle, kernel.encode(), ctypes.byref(ms), ctypes.byref(n),
             ctypes.byref(b))
        return ms.value, n.value, b.value

    @property
    def launches(self) -> int:
        n = c_uint64()
        call("tidq_ctx_launches", self.handle, ctypes.byref(n))
        return n.value


_contexts: dict[int, Context] = {}
_ctx_lock = threading.Lock()


_device_count: int | None = None


def device_count() -> int:
    """Visible CUDA devices (asked once per process: it cannot change)."""
    global _device_count
    if _device_count is None:
        n = c_int()
        call("tidq_device_count", ctypes.byref(n))
        _device_count = n.value
    return _device_count


def default_device() -> int:
    env = os.environ.get("TIDQ_DEVICE")
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0")) if device_count() > 1 else 0


def context(device: int | None = None) -> Context:
    """The process-wide context for ``device`` (created on first use)."""
    if device is None:
        device = default_device()
    ctx = _contexts.get(device)
    if ctx is None:
        with _ctx_lock:
            ctx = _contexts.get(device)
            if ctx is None:
                if device_count() == 0:
                    raise RuntimeError("no CUDA device visible: libtidq has no CPU fallback")
                ctx = Context(device)
                _contexts[device] = ctx
    return ctx


def total_launches() -> int:
    return sum(c.launches for c in _contexts.values())


# ---- device tables -------------------------------------------------------------


class DeviceTable:
    """Owner of a tidq_table handle: equal-length typed device columns."""

    __slots__ = ("handle", "_n", "_dtypes")

    def __init__(self, handle: c_void_p):
        self.handle = handle
        self._n = None  # resolved on first use: a TIDQ_SCAN_ASYNC result may still be in flight
        self._dtypes = None  # resolved on first use (two C calls per column saved per query)

    @property
    def dtypes(self) -> list:
        if self._dtypes is None:
            nc = c_int32()
            call("tidq_table_ncols", self.handle, ctypes.byref(nc))
            dts = []
            for k in range(nc.value):
                dt = c_int32()
                call("tidq_table_col_dtype", self.handle, k, ctypes.byref(dt))
                dts.append(DTYPES[dt.value])
            self._dtypes = dts
        return self._dtypes

    @property
    def n_rows(self) -> int:
        if self._n is None:
            n = c_uint64()
            call("tidq_table_info", self.handle, ctypes.byref(n), None)
            self._n = n.value
        return self._n

    @property
    def n_cols(self) -> int:
        return len(self.dtypes)

    def column(self, k: int) -> np.ndarray:
        out = pinned_empty(self.n_rows, self.dtypes[k])
        if self._n:
            call("tidq_table_download_col", self.handle, k, ptr(out))
        return out

    def free(self) -> None:
        if self.handle is not None and self.handle.value:
            call("tidq_table_free", self.handle)
        self.handle = None

    def __del__(self):
        try:
            if self.handle is not None and self.handle.value and _lib is not None:
                _lib.tidq_table_free(self.handle)
        except Exception:
            pass

    @classmethod
    def upload_u32(cls, ctx: Context, columns: list[np.ndarray]) -> "DeviceTable":
        cols = [np.ascontiguousarray(c, dtype=np.uint32) for c in columns]
        n = len(cols[0]) if cols else 0
        arr = (c_void_p * max(len(cols), 1))(*[ptr(c) for c in cols])
        h = c_void_p()
        call("tidq_table_upload_u32", ctx.handle, len(cols), arr, n, ctypes.byref(h))
        return cls(h)


def empty_spec() -> ScanSpec:
    return ScanSpec()


def run_scan(target, spec: ScanSpec, *, host=None) -> list[DeviceTable]:
    """Run one scan pass; ``target`` is a store handle, or a ctx when ``host``
    = (aos ndarray, n_triples, base_index) for the host-buffer variant."""
    out = (c_void_p * spec.n_streams)()
    if host is None:
        call("tidq_scan", target, ctypes.byref(spec), out)
    else:
        aos, n, base = host
        call("tidq_scan_host", target, ptr(aos), n, base, ctypes.byref(spec), out)
    return [DeviceTable(c_void_p(out[i])) for i in range(spec.n_streams)]
