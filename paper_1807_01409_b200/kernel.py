"""Drop-in for reference ``tripleid.kernel`` on the B200 scan kernel.

Same names, signatures, result types and errors as kernel.py:33-266:

- ``search_chunk(chunk, key, workers=1, *, write_counts=None) -> MatchResult``
  (int64 ascending global indices, uint8 answer codes)       kernel.py:148-179
- ``search_multi(chunk, keys, workers=1, *, write_counts=None) -> MatchResult``
  (int64 ascending global indices, uint32 mark sets)         kernel.py:182-227
- ``search_file(path, keys, workers=1, chunk_triples=None)``  kernel.py:230-254
- ``gather_rows(chunks, result)``                              kernel.py:257-266

``chunk`` may be a host ``TripleChunk`` (ours or the reference's: anything with
``.data`` and ``.base_index``) — uploaded, scanned and downloaded per call — or
a resident :class:`~paper_1807_01409_b200.store.DeviceStore` (no PCIe traffic
for the data).  ``workers`` is validated and otherwise ignored: the CUDA grid
replaces the thread pool (kernel.py:99-132) and results are worker-invariant
by contract.  ``write_counts`` keeps its instrumentation meaning:
the mark kernels themselves add 1 (device atomics) to the counter of every
triple slot they write, and the counters are added into the caller's array —
a test of write disjointness measures the real kernel.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from .errors import TooManySubqueries
from .store import ID_DTYPE, DeviceStore, TripleChunk, read_chunks

__all__ = [
    "MAX_SUBQUERIES",
    "TILE_TRIPLES",
    "ANSWER_LABELS",
    "TooManySubqueries",
    "PatternKey",
    "match_bits",
    "accepts",
    "MatchResult",
    "tile_spans",
    "search_chunk",
    "search_multi",
    "search_file",
    "gather_rows",
]

MAX_SUBQUERIES = 32
TILE_TRIPLES = 1 << 16  # reference CPU tile; the device tile is 4096 triples

ANSWER_LABELS = {7: "SPO", 6: "SP?", 5: "S?O", 4: "S??", 3: "?PO", 2: "?P?", 1: "??O", 0: "none"}


@dataclass(frozen=True, slots=True)
class PatternKey:
    subj: int = 0
    pred: int = 0
    obj: int = 0

    @property
    def bound_mask(self) -> int:
        return (4 if self.subj else 0) | (2 if self.pred else 0) | (1 if self.obj else 0)


def match_bits(triple: Sequence[int], key) -> int:
    s, p, o = triple
    return (4 if s == key.subj else 0) | (2 if p == key.pred else 0) | (1 if o == key.obj else 0)


def accepts(bits: int, key) -> bool:
    m = key.bound_mask
    return (bits & m) == m


@dataclass(frozen=True)
class MatchResult:
    indices: np.ndarray
    values: np.ndarray

    def __len__(self) -> int:
        return len(self.indices)


def tile_spans(n_triples: int, workers: int, tile: int = TILE_TRIPLES) -> list[list[tuple[int, int]]]:
    """Round-robin tile assignment of the reference CPU path (kernel.py:99-107);
    kept for API compatibility only."""
    spans: list[list[tuple[int, int]]] = [[] for _ in range(workers)]
    for t, lo in enumerate(range(0, n_triples, tile)):
        spans[t % workers].append((lo, min(lo + tile, n_triples)))
    return spans


def _key_ids(key) -> tuple[int, int, int]:
    return int(key.subj), int(key.pred), int(key.obj)


def _check_workers(workers: int) -> None:
    if workers < 1:
        raise ValueError("workers must be >= 1")


def _scan(chunk, spec: _lib.ScanSpec) -> list[_lib.DeviceTable]:
    if isinstance(chunk, DeviceStore):
        return _lib.run_scan(chunk.handle, spec)
    data = np.ascontiguousarray(chunk.data, dtype=ID_DTYPE).reshape(-1)
    n = data.size // 3
    ctx = _lib.context()
    return _lib.run_scan(ctx.handle, spec, host=(data, n, int(chunk.base_index)))


def _count(chunk) -> int:
    return chunk.triple_count


def _attach_write_counts(spec: _lib.ScanSpec, chunk, write_counts):
    """write_counts instrumentation (kernel.py:153,172-173,221-222): the mark
    kernels add 1 to the device counter of every triple slot they write; the
    counts are added into the caller's array after the scan."""
    if write_counts is None:
        return None
    wc = np.zeros(_count(chunk), dtype=np.uint32)
    spec.write_counts = wc.ctypes.data if wc.size else None
    spec._wc_keepalive = wc
    return wc


def search_chunk(chunk, key, workers: int = 1, *, write_counts: np.ndarray | None = None) -> MatchResult:
    """Accepted triples of one key with their answer codes (kernel.py:148-179)."""
    _check_workers(workers)
    spec = _lib.ScanSpec()
    spec.n_keys = 1
    spec.keys[0][:] = _key_ids(key)
    spec.n_streams = 1
    st = spec.streams[0]
    st.select = 1
    st.n_out = 2
    st.out[0] = _lib.OUT_INDEX
    st.out[1] = _lib.OUT_ANSWER
    st.answer_key = 0
    wc = _attach_write_counts(spec, chunk, write_counts)
    (table,) = _scan(chunk, spec)
    try:
        res = MatchResult(table.column(0), table.column(1))
    finally:
        table.free()
    if wc is not None:
        write_counts[: len(wc)] += wc
    return res


def search_multi(chunk, keys: Sequence, workers: int = 1, *,
                 write_counts: np.ndarray | None = None) -> MatchResult:
    """Mark sets of up to 32 keys in one pass (kernel.py:182-227)."""
    _check_workers(workers)
    keys = list(keys)
    if not 1 <= len(keys) <= MAX_SUBQUERIES:
        raise TooManySubqueries(f"{len(keys)} keys; supported range is 1..{MAX_SUBQUERIES}")
    spec = _lib.ScanSpec()
    spec.n_keys = len(keys)
    for q, k in enumerate(keys):
        spec.keys[q][:] = _key_ids(k)
    spec.n_streams = 1
    st = spec.streams[0]
    st.select = (1 << len(keys)) - 1
    st.n_out = 2
    st.out[0] = _lib.OUT_INDEX
    st.out[1] = _lib.OUT_MARKS
    wc = _attach_write_counts(spec, chunk, write_counts)
    (table,) = _scan(chunk, spec)
    try:
        res = MatchResult(table.column(0), table.column(1))
    finally:
        table.free()
    if wc is not None:
        write_counts[: len(wc)] += wc
    return res


def search_file(path, keys, workers: int = 1, chunk_triples: int | None = None) -> MatchResult:
    """Chunked search over a .tid file; chunk-size invariant (kernel.py:230-254)."""
    single = isinstance(keys, PatternKey) or (
        hasattr(keys, "subj") and hasattr(keys, "pred") and hasattr(keys, "obj")
    )
    parts = []
    # results are chunk-size invariant: a file that fits in HBM
    # is loaded whole by the native reader and scanned once
    if chunk_triples is not None and chunk_triples < 1:  # read_chunks' check comes first
        raise ValueError("chunk_triples must be >= 1")
    chunks = [DeviceStore.load(path)] if DeviceStore.fits(path) else read_chunks(path, chunk_triples)
    for chunk in chunks:
        parts.append(search_chunk(chunk, keys, workers) if single else search_multi(chunk, keys, workers))
    if not parts:
        return MatchResult(np.empty(0, dtype=np.int64),
                           np.empty(0, dtype=np.uint8 if single else np.uint32))
    return MatchResult(np.concatenate([p.indices for p in parts]),
                       np.concatenate([p.values for p in parts]))


def gather_rows(chunks: Iterable, result: MatchResult) -> np.ndarray:
    """Triple rows of a result's global indices, in result order (kernel.py:257-266)."""
    out = np.empty((len(result.indices), 3), dtype=ID_DTYPE)
    for chunk in chunks:
        lo = int(chunk.base_index)
        hi = lo + chunk.triple_count
        sel = (result.indices >= lo) & (result.indices < hi)
        if not sel.any():
            continue
        if isinstance(chunk, DeviceStore):
            out[sel] = chunk.gather(result.indices[sel] - lo)
        else:
            out[sel] = chunk.rows[result.indices[sel] - lo]
    return out
