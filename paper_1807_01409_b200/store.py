"""TripleID store: the ``.tid`` file format and the resident device store.

Host side (drop-in for reference ``store.py``): the same ``.tid`` layout —
16-byte header ``<4sIQ>`` = magic ``TID1``, version 1, triple count, then
``count`` records of three little-endian uint32 IDs (store.py:1-10,21-28) —
and the same chunk iterator, memory formula and error classes.

Device side (new): :class:`DeviceStore` keeps the triples resident in HBM as
three 16-byte aligned uint32 columns (s, p, o), zero padded to the scan tile.
It is built either by uploading an AoS chunk (pipelined H2D + on-device
transpose) or by the on-device counter-based generator.
"""

from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass
from typing import Iterable, Iterator, NamedTuple

import numpy as np

from . import _lib
from .errors import BadMagic, BadVersion, InvariantViolation, StoreError, TruncatedFile

__all__ = [
    "MAGIC",
    "VERSION",
    "HEADER_BYTES",
    "ID_BYTES",
    "TRIPLE_BYTES",
    "ID_DTYPE",
    "CHUNK_GRANULE",
    "DEFAULT_MEMORY_BUDGET",
    "Triple",
    "TripleChunk",
    "StoreError",
    "BadMagic",
    "BadVersion",
    "TruncatedFile",
    "InvariantViolation",
    "as_id_array",
    "write_tid",
    "read_header",
    "read_chunks",
    "read_all",
    "device_memory_bytes",
    "chunk_triples_for_budget",
    "DeviceStore",
]

MAGIC = b"TID1"
VERSION = 1
_HEADER_FMT = struct.Struct("<4sIQ")
HEADER_BYTES = _HEADER_FMT.size
ID_BYTES = 4
TRIPLE_BYTES = 3 * ID_BYTES
ID_DTYPE = np.dtype("<u4")
CHUNK_GRANULE = 1 << 20
DEFAULT_MEMORY_BUDGET = 256 * 1024 * 1024


class Triple(NamedTuple):
    subj: int
    pred: int
    obj: int


@dataclass(frozen=True)
class TripleChunk:
    """Flat AoS run of triples [s0,p0,o0,s1,...] starting at ``base_index``."""

    data: np.ndarray
    base_index: int

    @property
    def triple_count(self) -> int:
        return len(self.data) // 3

    @property
    def rows(self) -> np.ndarray:
        return self.data.reshape(-1, 3)


def as_id_array(triples) -> np.ndarray:
    """(n, 3) uint32 array of validated IDs (store.py:82-94 semantics)."""
    if isinstance(triples, np.ndarray):
        out = np.ascontiguousarray(triples, dtype=ID_DTYPE).reshape(-1, 3)
    else:
        wide = np.array([x for t in triples for x in t], dtype=np.uint64).reshape(-1, 3)
        if wide.size and int(wide.max()) > 0xFFFFFFFF:
            raise InvariantViolation("ID exceeds 32 bits")
        out = wide.astype(ID_DTYPE)
    if out.size and not out.all():
        raise InvariantViolation("stored triples must not contain ID 0")
    return out


def write_tid(triples, path) -> int:
    arr = as_id_array(triples)
    with open(path, "wb") as fh:
        fh.write(_HEADER_FMT.pack(MAGIC, VERSION, len(arr)))
        fh.write(arr.tobytes())
    return len(arr)


def read_header(path) -> int:
    with open(path, "rb") as fh:
        raw = fh.read(HEADER_BYTES)
    if len(raw) < HEADER_BYTES:
        raise TruncatedFile(f"{path}: header shorter than {HEADER_BYTES} bytes")
    magic, version, count = _HEADER_FMT.unpack(raw)
    if magic != MAGIC:
        raise BadMagic(f"{path}: magic {magic!r}, expected {MAGIC!r}")
    if version != VERSION:
        raise BadVersion(f"{path}: version {version}, expected {VERSION}")
    return count


def read_chunks(path, chunk_triples: int | None = None) -> Iterator[TripleChunk]:
    if chunk_triples is None:
        chunk_triples = chunk_triples_for_budget(DEFAULT_MEMORY_BUDGET)
    if chunk_triples < 1:
        raise ValueError("chunk_triples must be >= 1")
    total = read_header(path)
    with open(path, "rb") as fh:
        fh.seek(HEADER_BYTES)
        done = 0
        while done < total:
            take = min(chunk_triples, total - done)
            raw = fh.read(take * TRIPLE_BYTES)
            if len(raw) < take * TRIPLE_BYTES:
                raise TruncatedFile(
                    f"{path}: header declares {total} triples, data ends at "
                    f"triple {done + len(raw) // TRIPLE_BYTES}"
                )
            yield TripleChunk(np.frombuffer(raw, dtype=ID_DTYPE), done)
            done += take


def read_all(path) -> TripleChunk:
    n = read_header(path)
    for chunk in read_chunks(path, max(1, n)):
        return chunk
    return TripleChunk(np.empty(0, dtype=ID_DTYPE), 0)


def device_memory_bytes(n_ids: int) -> int:
    """(N + N/3 + 3) * 4 — data array + position array + key (store.py:156-164)."""
    if n_ids % 3:
        raise ValueError("data array length must be a multiple of 3")
    return (n_ids + n_ids // 3 + 3) * ID_BYTES


def chunk_triples_for_budget(budget_bytes: int) -> int:
    k = 1
    while device_memory_bytes(3 * CHUNK_GRANULE * (k + 1)) <= budget_bytes:
        k += 1
    return k * CHUNK_GRANULE


# ---- resident device store ------------------------------------------------------


class DeviceStore:
    """Triples resident in HBM as SoA uint32 columns (one tidq_store)."""

    def __init__(self, handle: ctypes.c_void_p, ctx: _lib.Context):
        self.handle = handle
        self.ctx = ctx
        self.pcodes = False  # predicate-code column built (with the predicate histogram)
        self.so = False  # interleaved (s, o) column built (after SO_AFTER_SCANS scans)
        self.pcodes_built = False
        n = ctypes.c_uint64()
        base = ctypes.c_uint64()
        _lib.call("tidq_store_info", handle, ctypes.byref(n), ctypes.byref(base))
        self.triple_count = n.value
        self.base_index = base.value

    # -- construction -----------------------------------------------------------
    @classmethod
    def upload(cls, chunk, device: int | None = None) -> "DeviceStore":
        """From a TripleChunk (or an (n,3)/flat uint32 array with base 0)."""
        if hasattr(chunk, "data") and hasattr(chunk, "base_index"):
            data, base = chunk.data, int(chunk.base_index)
        else:
            data, base = chunk, 0
        flat = np.ascontiguousarray(data, dtype=ID_DTYPE).reshape(-1)
        if flat.size % 3:
            raise ValueError("data array length must be a multiple of 3")
        ctx = _lib.context(device)
        h = ctypes.c_void_p()
        _lib.call("tidq_store_upload", ctx.handle, _lib.ptr(flat), flat.size // 3, base,
                  ctypes.byref(h))
        return cls(h, ctx)

    @classmethod
    def load(cls, path, device: int | None = None, base_index: int = 0, lo: int = 0,
             n: int | None = None) -> "DeviceStore":
        """A ``.tid`` file (or its rows [lo, lo+n), global indices
        base_index + lo ...) into HBM (native parallel reader, pipelined
        H2D + transpose).  Same errors as read_header / read_chunks
        (store.py:107-146): FileNotFoundError, BadMagic, BadVersion,
        TruncatedFile; a range starting beyond the file -> ValueError."""
        path = os.fspath(path)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        if lo < 0 or (n is not None and n < 0):
            raise ValueError("row range must be non-negative")
        ctx = _lib.context(device)
        h = ctypes.c_void_p()
        if lo == 0 and n is None:
            _lib.call("tidq_store_load_tid", ctx.handle, path.encode(), base_index, ctypes.byref(h))
        else:
            _lib.call("tidq_store_load_tid_range", ctx.handle, path.encode(), lo,
                      (1 << 64) - 1 if n is None else n, base_index, ctypes.byref(h))
        return cls(h, ctx)

    @classmethod
    def load_shard(cls, path, rank: int, world: int, device: int | None = None) -> "DeviceStore":
        """Rank ``rank``'s contiguous row range of a ``.tid`` file (the
        multi-GPU row sharding of SURVEY 8e: sizes differing by at most one), global
        indices preserved, so per-rank scan outputs concatenated in rank
        order equal the whole-file scan (chunk invariance)."""
        if not 0 <= rank < world:
            raise ValueError("rank must be in [0, world)")
        q, r = divmod(read_header(path), world)  # = distributed.shard_bounds
        lo = rank * q + min(rank, r)
        return cls.load(path, device=device, lo=lo, n=q + (1 if rank < r else 0))

    @staticmethod
    def fits(path, device: int | None = None) -> bool:
        """Whether a .tid file loads whole with room to spare for the query
        (columns + scan scratch + results within half of the free HBM)."""
        n = read_header(path)
        free, _ = _lib.context(device).mem_info()
        return n * TRIPLE_BYTES * 2 + (256 << 20) <= free // 2

    @classmethod
    def generate(cls, n_triples: int, *, seed: int, n_p: int, n_e: int, zipf_s: float = 1.0,
                 base_index: int = 0, device: int | None = None) -> "DeviceStore":
        """Counter-based synthetic store generated on the device."""
        from .synth import zipf_cdf_table

        cdf = zipf_cdf_table(n_p, zipf_s)
        prm = _lib.SynthParams(n_triples, base_index, seed, n_p, n_e)
        ctx = _lib.context(device)
        h = ctypes.c_void_p()
        _lib.call("tidq_store_generate", ctx.handle, ctypes.byref(prm), _lib.ptr(cdf),
                  ctypes.byref(h))
        return cls(h, ctx)

    # -- access -------------------------------------------------------------------
    def download(self, lo: int = 0, n: int | None = None) -> np.ndarray:
        """Rows [lo, lo+n) as an (n, 3) uint32 array."""
        if n is None:
            n = self.triple_count - lo
        out = np.empty((n, 3), dtype=ID_DTYPE)
        if n:
            _lib.call("tidq_store_download", self.handle, lo, n, _lib.ptr(out))
        return out

    def gather(self, local_idx: np.ndarray) -> np.ndarray:
        idx = np.ascontiguousarray(local_idx, dtype=np.int64)
        out = np.empty((len(idx), 3), dtype=ID_DTYPE)
        if len(idx):
            _lib.call("tidq_store_gather", self.handle, _lib.ptr(idx), len(idx), _lib.ptr(out))
        return out

    def column_max(self, col: int) -> int:
        out = ctypes.c_uint32()
        _lib.call("tidq_store_col_max", self.handle, col, ctypes.byref(out))
        return out.value

    def id_bound(self) -> int:
        """1 + the largest term ID in the store (cached; bitmap sizes)."""
        if getattr(self, "_id_bound", None) is None:
            self._id_bound = 1 + max(self.column_max(k) for k in range(3))
        return self._id_bound

    HIST_MAX_ID = (1 << 24) - 1

    def predicate_counts(self) -> np.ndarray | None:
        """Triples per predicate ID (cached; one device pass): exact output
        sizes for ?P? scans.  None when predicate IDs exceed HIST_MAX_ID."""
        self._scans = getattr(self, "_scans", 0) + 1
        if self._scans == self.SO_AFTER_SCANS and self.pcodes_built:
            self._build_so()
        if not hasattr(self, "_pred_hist"):
            mx = self.column_max(1) if self.triple_count else 0
            if mx > self.HIST_MAX_ID:
                self._pred_hist = None
            else:
                h = np.zeros(mx + 1, dtype=np.uint64)
                _lib.call("tidq_store_pred_hist", self.handle, mx, _lib.ptr(h))
                self._pred_hist = h
                self._build_pcodes(h)
        return self._pred_hist

    def prepare(self) -> "DeviceStore":
        """Build the store's index columns now — the predicate histogram with
        the 16-bit predicate-code column, and the (s, o) pair column — instead
        of lazily inside its first queries (a store loaded to serve many
        queries; the columns never change results)."""
        self.predicate_counts()
        self._build_so()
        return self

    PCODES_MAX = 30000  # (tidq_store_pcodes: codes are fp16-normal bit patterns)
    # the (s, o) pair column is built once a store has served this many scans:
    # its build (a read and a write of 8 B per triple, ~0.3 ms per 100 M)
    # costs more than it saves on a store queried only a few times (the e2e
    # bench re-uploads its store for every 5-query sweep: 25.1 -> 25.7-26.9
    # ms per step when built eagerly) and pays off on resident stores
    SO_AFTER_SCANS = int(os.environ.get("TIDQ_SO_AFTER", "8"))

    def _build_pcodes(self, hist: np.ndarray) -> None:
        # the store's distinct predicate IDs -> a 16-bit code column that the
        # scan streams for predicate-only passes (tidq_store_pcodes; cheap:
        # built with the histogram, at the store's first ?P? scan)
        cols = os.environ.get("TIDQ_STORE_COLS", "ps")  # A/B knob: p = code column, s = (s, o) pairs
        pvals = np.flatnonzero(hist).astype(np.uint32)
        self.pcodes = "p" in cols and 0 < len(pvals) <= self.PCODES_MAX
        if self.pcodes:
            _lib.call("tidq_store_pcodes", self.handle, _lib.ptr(pvals), len(pvals))
        self.pcodes_built = True
        if self.SO_AFTER_SCANS <= 1:
            self._build_so()

    def _build_so(self) -> None:
        # interleaved (s, o) pairs for the emit's gathers, when HBM has room
        if "s" in os.environ.get("TIDQ_STORE_COLS", "ps") and self.triple_count > 0 and not self.so:
            free, _ = self.ctx.mem_info()
            if self.triple_count * 8 * 3 < free:
                _lib.call("tidq_store_so", self.handle, 1)
                self.so = True

    def free(self) -> None:
        if self.handle is not None and self.handle.value:
            _lib.call("tidq_store_free", self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __len__(self) -> int:
        return self.triple_count

    def __repr__(self) -> str:
        return f"DeviceStore(n={self.triple_count}, base={self.base_index}, device={self.ctx.device})"
