"""Drop-in for reference ``tripleid.query_ops`` on the B200.

Same names, signatures, semantics and errors as query_ops.py:36-455; the
integer work runs in libtidq:

- scan (one pass for ALL groups' keys, ≤32 per pass — the reference makes one
  pass per group, query_ops.py:275-278) with the pattern_table
  repeated-variable mask (query_ops.py:220-225) and projection to the
  variables' first slots fused into the scan epilogue;
- FILTER: the regex runs on the host over the distinct candidate IDs, exactly
  as query_ops.py:241-252 (np.unique -> decode -> re.search on str_form); the
  device computes the distinct IDs and applies the accepted-ID bitmap.  When a
  complete bitmap for (dictionary, regex) is cached it is fused into the scan
  epilogue instead;
- joins: the left-deep chain of join_group (query_ops.py:298-342) with the
  device sort-merge join (merge_join order: key, left row, right row);
- UNION: device concatenation, UNBOUND = 0 for absent columns;
- DISTINCT: device radix sort + adjacent dedup, first occurrence kept in
  first-occurrence order (query_ops.py:393-398).

Intermediates stay in HBM; only the final table is downloaded.  ``store`` may
be a .tid path, a TripleChunk, a list of chunks (uploaded chunk by chunk), a
resident :class:`DeviceStore`, or a list of DeviceStores.  Output row order
equals the reference's.
"""

from __future__ import annotations

import ctypes
import os
import re
import weakref
from dataclasses import dataclass, field
from time import perf_counter
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from .errors import DisconnectedPatterns, ResourceLimit
from .plan import SLOT_LETTERS, compile_group
from .store import ID_DTYPE, DeviceStore, TripleChunk, read_chunks

__all__ = [
    "UNBOUND",
    "DEFAULT_ROW_CAP",
    "DisconnectedPatterns",
    "ResourceLimit",
    "Relationship",
    "analyze_relationships",
    "BindingRelation",
    "build_relation",
    "merge_join",
    "BindingTable",
    "pattern_table",
    "str_form",
    "apply_filter",
    "scan_patterns",
    "join_group",
    "evaluate_group",
    "evaluate_union",
    "project_distinct",
    "decode_table",
    "QueryTimings",
    "evaluate_query",
    "DevTable",
]

UNBOUND = 0
DEFAULT_ROW_CAP = 10_000_000


# ----------------------------------------------------------------------------- host types


@dataclass(frozen=True)
class Relationship:
    i: int
    j: int
    rel_type: str
    variable: str


def analyze_relationships(patterns) -> list[Relationship]:
    """Pattern j joins the closest earlier pattern sharing a variable, on the
    shared variable with the smallest slot in pattern i (query_ops.py:63-91)."""
    if len(patterns) < 2:
        return []
    maps = [p.var_slots() for p in patterns]
    rels = []
    for j in range(1, len(patterns)):
        rel = None
        for i in range(j - 1, -1, -1):
            common = sorted((v for v in maps[i] if v in maps[j]), key=lambda v: maps[i][v][0])
            if common:
                v = common[0]
                rel = Relationship(i, j, SLOT_LETTERS[maps[i][v][0]] + SLOT_LETTERS[maps[j][v][0]], v)
                break
        if rel is None:
            raise DisconnectedPatterns(f"pattern {j} shares no variable with any earlier pattern")
        rels.append(rel)
    return rels


@dataclass
class BindingRelation:
    """query_ops.py:94-118 (API type; not used by join_group)."""

    key: np.ndarray
    values: dict
    sorted: bool = False

    def __len__(self) -> int:
        return len(self.key)

    def prepare_for_join(self) -> "BindingRelation":
        """Key sorted nondecreasing (stable), values permuted alike
        (query_ops.py:110-118); the sort runs on the device."""
        if self.sorted:
            return self
        key = np.ascontiguousarray(self.key, dtype=np.uint32)
        skey = np.empty(len(key), dtype=np.uint32)
        order = np.empty(len(key), dtype=np.uint32)
        if len(key):
            _lib.call("tidq_argsort_u32", _lib.context().handle, _lib.ptr(key), len(key), _lib.ptr(skey),
                      _lib.ptr(order))
        return BindingRelation(skey.astype(self.key.dtype, copy=False),
                               {k: np.asarray(v)[order] for k, v in self.values.items()}, True)


def build_relation(rows: np.ndarray, pattern, join_slot: str) -> BindingRelation:
    """query_ops.py:121-136."""
    idx = SLOT_LETTERS.index(join_slot)
    slot = pattern.slots[idx]
    name = slot.name if hasattr(slot, "name") else None
    if not pattern.var_slots().get(name):
        raise ValueError(f"join slot {join_slot} is not a variable of the pattern")
    rows = np.asarray(rows).reshape(-1, 3)
    return BindingRelation(rows[:, idx].copy(),
                           {SLOT_LETTERS[k]: rows[:, k].copy() for k in range(3) if k != idx})


@dataclass
class BindingTable:
    """Materialized solution rows: one uint32 column per variable."""

    columns: list
    data: dict = field(default_factory=dict)

    @classmethod
    def empty(cls, columns) -> "BindingTable":
        cols = list(columns)
        return cls(cols, {c: np.empty(0, dtype=ID_DTYPE) for c in cols})

    @property
    def n_rows(self) -> int:
        return len(self.data[self.columns[0]]) if self.columns else 0

    def take(self, indices) -> "BindingTable":
        return BindingTable(list(self.columns), {c: self.data[c][indices] for c in self.columns})

    def row_tuples(self) -> list:
        if not self.columns:
            return []
        st = np.stack([self.data[c] for c in self.columns], axis=1)
        return [tuple(int(x) for x in r) for r in st]


def str_form(lexical: str) -> str:
    """SPARQL str() of a term token (query_ops.py:232-238)."""
    if lexical.startswith("<"):
        return lexical[1:-1]
    if lexical.startswith('"'):
        return lexical[1:lexical.rfind('"')]
    return lexical


# ----------------------------------------------------------------------------- device tables


class DevTable:
    """Named device columns (uint32), the device twin of BindingTable."""

    __slots__ = ("columns", "t", "_n", "reduced", "keybm")

    def __init__(self, columns: list, t: _lib.DeviceTable | None, n_rows: int | None = None):
        self.columns = list(columns)
        self.t = t
        self.reduced = False  # semi-join reduced by the scan (_reduced_tables)
        self.keybm = None     # (variable, _DeviceBitmap): key set built by the scan's emit
        if not self.columns:
            self._n = 0  # a table without columns has no rows (query_ops.py:193-196)
        else:
            self._n = n_rows  # None: read from the device table on first use

    @property
    def n_rows(self) -> int:
        if self._n is None:
            self._n = self.t.n_rows
        return self._n

    def col(self, name: str) -> int:
        return self.columns.index(name)

    def download(self) -> BindingTable:
        if not self.columns:
            return BindingTable([], {})
        return BindingTable(list(self.columns), {c: self.t.column(k) for k, c in enumerate(self.columns)})

    @classmethod
    def upload(cls, columns: list, data: dict, ctx=None) -> "DevTable":
        ctx = ctx or _lib.context()
        return cls(columns, _lib.DeviceTable.upload_u32(ctx, [np.asarray(data[c]) for c in columns]))

    @classmethod
    def from_handle(cls, columns, h: ctypes.c_void_p) -> "DevTable":
        return cls(columns, _lib.DeviceTable(h))


def _new_handle(fn: str, *args) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _lib.call(fn, *args, ctypes.byref(h))
    return h


def _i32(xs) -> ctypes.Array:
    return (ctypes.c_int32 * max(len(xs), 1))(*xs)


def _dev_concat(ctx, tables: list[DevTable], columns: list) -> DevTable:
    tables = [t for t in tables if t.columns]  # column-less tables hold no rows
    src = []
    for t in tables:
        src += [t.col(c) if c in t.columns else -1 for c in columns]
    hs = (ctypes.c_void_p * max(len(tables), 1))(*[t.t.handle.value if t.t else None for t in tables])
    return DevTable.from_handle(columns, _new_handle("tidq_table_concat", ctx.handle, len(tables), hs,
                                                     len(columns), _i32(src)))


def _dev_project(t: DevTable, columns: list) -> DevTable:
    if columns == t.columns:
        return t
    idx = [t.col(c) for c in columns]
    return DevTable.from_handle(columns, _new_handle("tidq_table_project", t.t.handle, len(idx), _i32(idx)))


def _dev_distinct(t: DevTable, columns: list, key_bound: int = 0) -> DevTable:
    idx = [t.col(c) for c in columns]
    return DevTable.from_handle(columns, _new_handle("tidq_distinct_bound", t.t.handle, len(idx), _i32(idx),
                                                     int(key_bound)))


def _dev_filter_bitmap(t: DevTable, column: str, bitmap: "_DeviceBitmap") -> DevTable:
    return DevTable.from_handle(t.columns, _new_handle("tidq_table_filter_bitmap", t.t.handle,
                                                       t.col(column), bitmap.handle))


def _dev_unique(t: DevTable, column: str) -> np.ndarray:
    u = _lib.DeviceTable(_new_handle("tidq_table_unique_col", t.t.handle, t.col(column)))
    try:
        return u.column(0)
    finally:
        u.free()


class _ColRef(ctypes.Structure):
    _fields_ = [("side", ctypes.c_int32), ("col", ctypes.c_int32)]


JOIN_REDUCED = 1  # tidq.h TIDQ_JOIN_REDUCED


def _dev_join(left: DevTable, right: DevTable, var: str, row_cap, algo: int = 0, key_bound: int = 0) -> DevTable:
    """One step of the left-deep chain (query_ops.py:318-341)."""
    return _dev_join_counted(left, right, var, row_cap, algo, key_bound)[0]


def _key_bitmap(t: DevTable, var: str):
    """The scan-built key set of ``t`` on ``var``, if any."""
    if t.keybm is not None and t.keybm[0] == var:
        return t.keybm[1].handle
    return None


def _dev_join_counted(left: DevTable, right: DevTable, var: str, row_cap, algo: int = 0,
                      key_bound: int = 0) -> tuple:
    """_dev_join plus the merge-join pair count (before the equality mask)."""
    cols = list(left.columns)
    refs = [(0, k) for k in range(len(left.columns))]
    eq = []
    for k, c in enumerate(right.columns):
        if c == var:
            continue
        if c in cols:
            eq += [left.col(c), k]
        else:
            cols.append(c)
            refs.append((1, k))
    arr = (_ColRef * max(len(refs), 1))(*[_ColRef(s, k) for s, k in refs])
    n_pairs = ctypes.c_uint64()
    h = ctypes.c_void_p()
    cap = -1 if row_cap is None else int(row_cap)
    lbm, rbm = (_key_bitmap(left, var), _key_bitmap(right, var)) if key_bound else (None, None)
    _lib.call("tidq_join", left.t.handle, left.col(var), right.t.handle, right.col(var), len(refs), arr,
              len(eq) // 2, _i32(eq), cap, algo, key_bound, lbm, rbm, ctypes.byref(h), ctypes.byref(n_pairs))
    return DevTable.from_handle(cols, h), n_pairs.value


# ----------------------------------------------------------------------------- FILTER


class _DeviceBitmap:
    def __init__(self, ctx, words: np.ndarray | None, n_bits: int):
        self.ctx = ctx
        if words is None:  # all zero, created on the device
            self.handle = _new_handle("tidq_bitmap_create", ctx.handle, n_bits)
        else:
            self.handle = _new_handle("tidq_bitmap_upload", ctx.handle, _lib.ptr(words), n_bits)

    def __del__(self):
        try:
            if self.handle and self.handle.value and _lib._lib is not None:
                _lib._lib.tidq_bitmap_free(self.handle)
        except Exception:
            pass


_PARALLEL_MIN = 200_000  # distinct IDs before the regex fans out to host cores
_worker_state: dict = {}  # set once per forked worker by _regex_worker_init (never in the parent)


def _regex_search(rx, dictionary, ids: np.ndarray) -> np.ndarray:
    return np.fromiter((bool(rx.search(str_form(dictionary.decode_lexical(int(u))))) for u in ids.tolist()),
                       dtype=bool, count=len(ids))


def _regex_worker_init(rx, dictionary, ids) -> None:
    _worker_state.update(rx=rx, d=dictionary, ids=ids)


def _regex_span(span) -> np.ndarray:
    lo, hi = span
    return _regex_search(_worker_state["rx"], _worker_state["d"], _worker_state["ids"][lo:hi])


def _regex_hits(rx, dictionary, ids: np.ndarray) -> np.ndarray:
    """re.search(str_form(decode(id))) for every id — Python ``re``, exactly
    the reference's predicate (query_ops.py:245-250).  Large ID sets are split
    over forked worker processes (the host side of FILTER is string work; the
    GIL rules out threads).  The workers receive the regex, dictionary and IDs
    as fork-inherited initializer arguments — nothing is parked in module
    state of the calling process, so concurrent FILTERs do not interfere — and
    never touch the CUDA context they inherit."""
    n = len(ids)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    if n < _PARALLEL_MIN or cores < 2:
        return _regex_search(rx, dictionary, ids)
    import multiprocessing as mp
    import warnings

    step = -(-n // (cores * 4))
    spans = [(lo, min(n, lo + step)) for lo in range(0, n, step)]
    with warnings.catch_warnings():
        # the parent holds CUDA/driver threads; the children only run Python re
        warnings.simplefilter("ignore", DeprecationWarning)
        with mp.get_context("fork").Pool(cores, initializer=_regex_worker_init,
                                         initargs=(rx, dictionary, ids)) as pool:
            parts = pool.map(_regex_span, spans)
    return np.concatenate(parts)


class _RegexCache:
    """Per (dictionary, regex): which IDs were tested and which matched.

    The regex itself always runs on the host with Python ``re`` on
    ``str_form(dictionary.decode_lexical(id))`` — identical semantics to
    query_ops.py:245-250 — but each ID is evaluated once per dictionary."""

    def __init__(self, regex: str):
        self.rx = re.compile(regex)
        self.tested = np.zeros(0, dtype=np.uint32)
        self.accepted = np.zeros(0, dtype=np.uint32)
        self.complete_upto = 0  # every ID in 1..complete_upto tested
        self._dev: dict = {}

    def _grow(self, max_id: int) -> None:
        words = (max_id >> 5) + 1
        if words > len(self.tested):
            for name in ("tested", "accepted"):
                old = getattr(self, name)
                new = np.zeros(max(words, 2 * len(old)), dtype=np.uint32)
                new[: len(old)] = old
                setattr(self, name, new)

    def evaluate(self, ids: np.ndarray, dictionary) -> None:
        if not len(ids):
            return
        self._grow(int(ids.max()))
        w, b = ids >> 5, (ids & 31).astype(np.uint32)
        new = ids[((self.tested[w] >> b) & 1) == 0]
        if len(new):
            hits = _regex_hits(self.rx, dictionary, new)
            nw, nb = new >> 5, (new & 31).astype(np.uint32)
            np.bitwise_or.at(self.tested, nw, np.uint32(1) << nb)
            acc = new[hits]
            if len(acc):
                np.bitwise_or.at(self.accepted, acc >> 5, np.uint32(1) << (acc & 31).astype(np.uint32))
            self._dev.clear()

    def evaluate_all(self, max_id: int, dictionary) -> None:
        """Evaluate every ID 1..max_id (in parallel) and mark the cache
        complete, so scans can fuse this FILTER as a bitmap test.  Only IDs
        above the previous ``complete_upto`` are evaluated (a dictionary that
        grew, e.g. by run_rule's encode_lexical, extends the bitmap)."""
        lo = self.complete_upto + 1
        if max_id < lo:
            return
        self._grow(max_id)
        ids = np.arange(lo, max_id + 1, dtype=np.uint32)
        hits = _regex_hits(self.rx, dictionary, ids)
        for name, mask in (("tested", np.ones(len(ids), dtype=bool)), ("accepted", hits)):
            words = getattr(self, name)
            # bits lo..max_id: whole words via packbits, the partial first word by OR
            first = (lo + 31) >> 5 << 5  # first word-aligned ID >= lo
            head = min(first, max_id + 1) - lo
            for k in np.nonzero(mask[:head])[0]:
                i = lo + int(k)
                words[i >> 5] |= np.uint32(1 << (i & 31))
            rest = mask[head:]
            if len(rest):
                packed = np.packbits(rest, bitorder="little")
                pad = np.zeros(-(-len(rest) // 32) * 4, dtype=np.uint8)
                pad[: len(packed)] = packed
                w0 = first >> 5
                seg = pad.view(np.uint32)
                words[w0: w0 + len(seg)] |= seg
        self.complete_upto = max_id
        self._dev.clear()

    def device_bitmap(self, ctx) -> _DeviceBitmap:
        bm = self._dev.get(ctx.device)
        if bm is None:
            bm = _DeviceBitmap(ctx, self.accepted, len(self.accepted) * 32)
            self._dev[ctx.device] = bm
        return bm


_regex_caches: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_regex_caches_by_id: dict = {}


def _cache_for(dictionary, regex: str) -> _RegexCache:
    try:
        per = _regex_caches.setdefault(dictionary, {})
    except TypeError:  # not weak-referenceable
        per = _regex_caches_by_id.setdefault(id(dictionary), {})
    c = per.get(regex)
    if c is None:
        c = per[regex] = _RegexCache(regex)
    return c


FULL_FILTER_MAX_ID = 1 << 27  # dictionaries up to 134M terms get a complete bitmap


def _dictionary_max_id(dictionary) -> int | None:
    mx = getattr(dictionary, "max_id", None)
    if mx is None:
        try:
            mx = len(dictionary)  # reference Dictionary: dense IDs 1..len (dictionary.py:64-69)
        except TypeError:
            return None
    return int(mx)


def prepare_filter(dictionary, regex: str, max_id: int | None = None) -> None:
    """Evaluate ``regex`` over every ID 1..max_id once (host cores in
    parallel), so scans fuse the FILTER as a bitmap test in the scan epilogue
    (no second pass, no per-query host regex)."""
    mx = _dictionary_max_id(dictionary) if max_id is None else int(max_id)
    if mx is None:
        raise ValueError("dictionary has no max_id; pass max_id")
    c = _cache_for(dictionary, regex)
    if c.complete_upto < mx:
        c.evaluate_all(mx, dictionary)


def _device_filter(t: DevTable, variable: str, regex: str, dictionary) -> DevTable:
    """apply_filter on a device table: distinct IDs on the device, regex on
    the host for unseen IDs, accepted-ID bitmap applied on the device."""
    cache = _cache_for(dictionary, regex)  # compiles: re.error as query_ops.py:245, even for no rows
    if t.n_rows == 0:
        return t
    cache.evaluate(_dev_unique(t, variable), dictionary)
    return _dev_filter_bitmap(t, variable, cache.device_bitmap(_lib.context()))


def apply_filter(table: BindingTable, variable: str, pattern: str, dictionary) -> BindingTable:
    """Keep rows whose term for ``variable`` matches the regex (query_ops.py:241-252)."""
    _cache_for(dictionary, pattern)  # re.error first, as the reference compiles first
    if variable not in table.data:
        raise KeyError(variable)  # table.data[variable] in the reference
    dt = DevTable.upload(table.columns, table.data)
    return _device_filter(dt, variable, pattern, dictionary).download()


# ----------------------------------------------------------------------------- scan


def _as_stores(store, chunk_triples):
    if isinstance(store, DeviceStore):
        return [store], False
    if isinstance(store, (list, tuple)) and store and all(isinstance(s, DeviceStore) for s in store):
        return list(store), False
    if isinstance(store, TripleChunk) or (hasattr(store, "data") and hasattr(store, "base_index")):
        return [store], True
    if isinstance(store, (list, tuple)):
        return list(store), True
    if chunk_triples is not None and chunk_triples < 1:  # read_chunks' check comes first
        raise ValueError("chunk_triples must be >= 1")
    if DeviceStore.fits(store):  # a .tid path: one native load, one scan (chunk-invariant)
        return [DeviceStore.load(store)], False
    return read_chunks(store, chunk_triples), True


def _live_columns(pattern, needed) -> list:
    """The pattern's variables the rest of the query reads (all when
    ``needed`` is None); at least one, so a table keeps its row count."""
    cols = pattern.variables()
    if needed is None:
        return cols
    live = [v for v in cols if v in needed]
    return live or cols[:1]


def _needed_variables(compiled, group) -> set | None:
    """Dead-column elimination: variables of ``group`` that the query reads
    after the scan — projected ones, join variables (shared by two patterns)
    and FILTER variables.  None = keep everything (SELECT *)."""
    if compiled is None or compiled.projection is None:
        return None
    need = set(compiled.projection)
    seen: dict = {}
    for pat in group.patterns:
        for v in pat.variables():
            seen[v] = seen.get(v, 0) + 1
    need |= {v for v, k in seen.items() if k > 1}
    need |= {f.variable for f in group.filters}
    return need


def _pattern_spec(pattern, var_slots, needed=None):
    """Outputs (first slot per live variable, in pattern.variables() order)
    and the repeated-variable equality flags of one pattern."""
    outs = [var_slots[v][0] for v in _live_columns(pattern, needed)]
    eq = 0
    for slots in var_slots.values():
        for extra in slots[1:]:
            pair = {slots[0], extra}
            eq |= _lib.EQ_SP if pair == {0, 1} else _lib.EQ_SO if pair == {0, 2} else _lib.EQ_PO
    return outs, eq


_IDX = "#idx"  # the scan column of local triple indices (semi-join reduced groups)


def _join_variables(group) -> list:
    """Join variables of a group worth reducing in the scan: those bound by
    two or more patterns, when some variable is bound by three or more (a
    star: the intersection of 3+ key sets is far more selective than the
    join's own pairwise pre-filter).  Measured on C4/C5: star x3/x4 and C5
    star x3 gain 9-15 %; two-pattern groups and chains lose 5-15 % (the
    reduction equals the join's own, plus the late gather), so they get [];
    so do groups with a FILTER, whose filtered table already shrinks the joins
    (star x3/x4 FILTER: 2.40 -> 2.51, 3.21 -> 3.34 ms when reduced)."""
    if group.filters:
        return []
    seen: dict = {}
    for pat in group.patterns:
        for v in pat.variables():
            seen[v] = seen.get(v, 0) + 1
    if not seen or max(seen.values()) < 3:
        return []
    return [v for v, k in seen.items() if k > 1]


# total bytes of emit-built join key sets per scan (above: the joins build
# their own); TIDQ_KEYSET_MAX_MB overrides for A/B measurements
_KEYSET_MAX_BYTES = int(os.environ.get("TIDQ_KEYSET_MAX_MB", "24")) << 20
# one gather pass for every pattern's deferred variables (TIDQ_GATHER_MULTI=0:
# one tidq_store_gather_cols per pattern, for A/B)
_GATHER_MULTI = os.environ.get("TIDQ_GATHER_MULTI", "1") != "0"
# late materialisation of join-free variables (TIDQ_DEFER=0 disables, for A/B)
_DEFER = os.environ.get("TIDQ_DEFER", "1") != "0"

_DEF = "#d"  # scan column of local triple indices standing in for pattern pj's deferred variables


def _deferred_variables(group, pj: int, live: list) -> list:
    """Variables of pattern ``pj`` the group's join chain never reads: bound
    by this pattern only (not a join key, not shared) and not FILTERed.  The
    scan emits the local triple index instead of gathering them, the joins
    carry the index, and _materialize gathers them for the group's result
    rows only (late materialisation; pair counts, row order and ResourceLimit
    are unchanged because every join key is still emitted)."""
    seen: dict = {}
    for pat in group.patterns:
        for v in pat.variables():
            seen[v] = seen.get(v, 0) + 1
    filtered = {f.variable for f in group.filters}
    return [v for v in live if seen.get(v, 0) == 1 and v not in filtered]


def _materialize(ds: DeviceStore, group, t: DevTable, needed) -> DevTable:
    """Replace each deferred-index column of a join result by the deferred
    variables it stands for (tidq_store_gather_cols, one launch per pattern),
    each call writing its columns in the order the chain produces without
    deferral, so the last one leaves exactly that order (no projection copy)."""
    expect: list = []
    for pat in [group.patterns[0]] + [group.patterns[r.j] for r in analyze_relationships(group.patterns)]:
        for v in _live_columns(pat, needed):
            if v not in expect:
                expect.append(v)
    if _GATHER_MULTI:  # every pattern's deferred variables in one pass, straight into the final order
        owner: dict = {}
        for pj, (pat, vs) in enumerate(zip(group.patterns, group.var_slots)):
            if f"{_DEF}{pj}" in t.columns:
                for v in _deferred_variables(group, pj, _live_columns(pat, needed)):
                    owner.setdefault(v, pj)
        spec, idx = [], []
        for v in expect:
            if v in t.columns:
                spec.append(t.col(v))
                idx.append(-1)
            elif v in owner:
                spec.append(-1 - group.var_slots[owner[v]][v][0])
                idx.append(t.col(f"{_DEF}{owner[v]}"))
            else:
                break
        else:
            if 0 < sum(1 for x in spec if x < 0) <= 8 and len(spec) <= 16:
                h = _new_handle("tidq_store_gather_cols_multi", ds.handle, t.t.handle, len(spec), _i32(spec),
                                _i32(idx))
                return DevTable.from_handle(expect, h)
    for pj, (pat, vs) in enumerate(zip(group.patterns, group.var_slots)):
        name = f"{_DEF}{pj}"
        if name not in t.columns:
            continue
        dv = _deferred_variables(group, pj, _live_columns(pat, needed))
        have = set(t.columns) | set(dv)
        cols = [c for c in expect if c in have] + [c for c in t.columns if c.startswith(_DEF) and c != name]
        spec = [t.col(c) if c in t.columns else -1 - vs[c][0] for c in cols]
        h = _new_handle("tidq_store_gather_cols", ds.handle, t.t.handle, t.col(name), len(spec), _i32(spec))
        t = DevTable.from_handle(cols, h)
    return _dev_project(t, expect)


def _scan_device(units, groups, dictionary, fuse_filters: bool, compiled=None, reduce: bool = True,
                 concat: bool = False, semijoin: bool = True, defer: bool = False):
    """Per group, per pattern: DevTable of the pattern's live variables
    (repeated variables checked, fused FILTERs applied), rows in ascending
    triple order.  ``units`` yields DeviceStores (or host chunks, uploaded one
    at a time).

    Groups with joins on a single resident store are scanned semi-join
    reduced (late materialisation): the scan emits only each pattern's join
    variables and its triple index; per join variable, every table keeps the
    rows whose value occurs in all other tables binding it
    (tidq_tables_semijoin — a row without such partners cannot be in the
    group's join, query_ops.py:298-342, and row order is kept); only then are
    the remaining columns gathered from the store for the survivors
    (tidq_store_gather_cols).  The join chain itself is unchanged.

    The reduction changes the pair counts of the chain's intermediate joins
    (rows that a later pattern would drop are gone before the first join), so
    it is only taken when no row cap is checked (``semijoin`` = row_cap is
    None): the reference raises ResourceLimit on the UNREDUCED pair count of
    every merge_join (query_ops.py:321-324).  The scan-built key sets below
    (each join's own pairwise pre-filter) keep every pair count unchanged.

    ``concat`` (a UNION of single-pattern groups with the same columns,
    _concat_union): one scan writes every group's rows into group 0's table
    in group order (TIDQ_SCAN_CONCAT); the other groups' tables are empty."""
    ctx = _lib.context()
    units = list(units)
    needed = [_needed_variables(compiled, g) for g in groups]
    single = len(units) == 1 and not units[0][1]
    # key bitmaps (semi-join reduction, scan-built key sets) are sized by the
    # store's largest ID: only for ID spaces up to 2^31 (256 MB per set)
    small_ids = single and units[0][0].id_bound() <= (1 << 31)
    jvars = [(_join_variables(g) if reduce and semijoin and small_ids and g.satisfiable and len(g.patterns) >= 2 else [])
             for g in groups]
    # late materialisation of the variables no join reads (one resident
    # store: the local indices must refer to it when the chain ends)
    dvars = [[(_deferred_variables(g, pj, _live_columns(pat, needed[gi]))
               if defer and _DEFER and single and not jvars[gi] and g.satisfiable and 2 <= len(g.patterns)
               and len({v for p in g.patterns for v in p.variables()}) <= 12 else [])
              for pj, pat in enumerate(g.patterns)] for gi, g in enumerate(groups)]
    # Key sets for the join chain, built by the scan's emit while each row is
    # in registers (a join otherwise builds both with a pass of atomics):
    # pattern 0 on the first relationship's variable, pattern j on its own.
    key_bits = units[0][0].id_bound() if small_ids and reduce else 0
    # ... only while the key sets of one scan stay small next to the L2
    # (C4, 2^26 IDs, 8 MB each: star/chain x2 2.02 -> 1.93 ms; C5, 2^28 IDs,
    # 3 x 32 MB: the emit's atomics and its gathers thrash L2, chain x3
    # 6.3 -> 6.9 ms)
    n_joins = sum(len(g.patterns) for g in groups if g.satisfiable and len(g.patterns) >= 2)
    if key_bits // 8 * n_joins > _KEYSET_MAX_BYTES:
        key_bits = 0
    keyvar: list = []
    for gi, g in enumerate(groups):
        kv = {}
        # (not under FILTER: the join's own key sets come from the filtered,
        # much smaller tables; measured 0.05-0.15 ms slower from the scan)
        if key_bits and not jvars[gi] and not g.filters and g.satisfiable and len(g.patterns) >= 2:
            try:
                rels = analyze_relationships(g.patterns)
            except DisconnectedPatterns:
                rels = []
            for k, rel in enumerate(rels):
                if k == 0:
                    kv[0] = rel.variable
                kv[rel.j] = rel.variable
        keyvar.append(kv)
    kbm: dict = {}
    # the largest ID of the resident stores (FILTER fusion needs a bitmap
    # covering it); host chunks take the unfused FILTER path
    resident_ids = None
    if fuse_filters and units and not any(host for _, host in units) and any(g.filters for g in groups):
        resident_ids = max(u.id_bound() for u, _ in units) - 1
    jobs = []  # (group index, pattern index, key, outs, eq, filters)
    for gi, g in enumerate(groups):
        if not g.satisfiable:
            continue
        for pj, (pat, vs, key) in enumerate(zip(g.patterns, g.var_slots, g.keys)):
            outs, eq = _pattern_spec(pat, vs, needed[gi])
            if jvars[gi]:  # reduced: local index + this pattern's join variables
                outs = [_lib.OUT_LOCAL] + [vs[v][0] for v in pat.variables() if v in jvars[gi]]
            else:
                if dvars[gi][pj]:  # deferred variables: their local triple index instead
                    outs = [vs[v][0] for v in _live_columns(pat, needed[gi]) if v not in dvars[gi][pj]] + [_lib.OUT_LOCAL]
                if keyvar[gi] and pj in keyvar[gi]:  # the join's key set, built by the emit
                    v = keyvar[gi][pj]
                    kbm[(gi, pj)] = (v, vs[v][0], _DeviceBitmap(ctx, None, key_bits))
            fused = []
            if fuse_filters and dictionary is not None and resident_ids is not None:
                for flt in g.filters:
                    if flt.variable in vs:
                        c = _cache_for(dictionary, flt.regex)
                        # (re-)read the dictionary's size: terms added since the
                        # bitmap was built (run_rule's encode_lexical, further
                        # conversions) are evaluated before the bitmap is fused
                        mx = _dictionary_max_id(dictionary)
                        if mx is not None and c.complete_upto < mx <= FULL_FILTER_MAX_ID:
                            c.evaluate_all(mx, dictionary)
                        # fused only when every ID the store holds was tested;
                        # otherwise the unfused path decodes (and raises on)
                        # unknown IDs exactly like query_ops.py:246-248
                        if c.complete_upto >= resident_ids and len(fused) < _lib.MAX_FILTERS:
                            fused.append((vs[flt.variable][0], c, flt))
            jobs.append((gi, pj, (int(key.subj), int(key.pred), int(key.obj)), outs, eq, fused))
    parts: dict = {}
    for unit, host in (units if jobs else ()):
        ds = DeviceStore.upload(unit) if host else unit
        try:
            for lo in range(0, len(jobs), _lib.MAX_STREAMS):
                batch = jobs[lo: lo + _lib.MAX_STREAMS]
                keys: list = []
                spec = _lib.ScanSpec()
                spec.n_streams = len(batch)
                for s, (gi, pj, key, outs, eq, fused) in enumerate(batch):
                    if key not in keys:
                        keys.append(key)
                    st = spec.streams[s]
                    st.select = 1 << keys.index(key)
                    st.eq_flags = eq
                    st.n_out = len(outs)
                    for k, slot in enumerate(outs):
                        st.out[k] = slot
                    st.n_filters = len(fused)
                    for f, (slot, cache, _flt) in enumerate(fused):
                        st.filter_slot[f] = slot
                        st.filter[f] = cache.device_bitmap(ctx).handle.value
                    if (gi, pj) in kbm:
                        st.key_bitmap = kbm[(gi, pj)][2].handle.value
                        st.key_bitmap_slot = kbm[(gi, pj)][1]
                spec.n_keys = len(keys)
                for q, key in enumerate(keys):
                    spec.keys[q][:] = key
                _capacity_hints(ds, spec, keys)
                if all(spec.streams[s].capacity_hint > 0 for s in range(spec.n_streams)):
                    spec.flags = _lib.SCAN_ASYNC  # histogram hints are exact bounds: do not wait
                    if concat and len(batch) == len(jobs):
                        spec.flags |= _lib.SCAN_CONCAT
                tables = _lib.run_scan(ds.handle, spec)
                for (gi, pj, *_), t in zip(batch, tables):
                    parts.setdefault((gi, pj), []).append(t)
        finally:
            if host:
                ds.free()
    out = []
    for gi, g in enumerate(groups):
        row = []
        if jvars[gi] and all((gi, pj) in parts for pj in range(len(g.patterns))):
            out.append(_reduced_tables(units[0][0], g, [parts[(gi, pj)][0] for pj in range(len(g.patterns))],
                                       jvars[gi], needed[gi]))
            continue
        for pj, pat in enumerate(g.patterns):
            cols = _live_columns(pat, needed[gi])
            if dvars[gi][pj]:
                cols = [v for v in cols if v not in dvars[gi][pj]] + [f"{_DEF}{pj}"]
            ts = parts.get((gi, pj), [])
            if not ts:
                row.append(DevTable.upload(cols, {c: np.empty(0, ID_DTYPE) for c in cols}, ctx))
            elif len(ts) == 1:
                row.append(DevTable(cols, ts[0]))
                if (gi, pj) in kbm:
                    row[-1].keybm = (kbm[(gi, pj)][0], kbm[(gi, pj)][2])
            else:
                row.append(_dev_concat(ctx, [DevTable(cols, t) for t in ts], cols))
        out.append(row)
    # FILTERs that were not fused: device distinct + host regex + device bitmap
    for gi, g in enumerate(groups):
        for flt in g.filters:
            for pj, pat in enumerate(g.patterns):
                if flt.variable not in pat.var_slots():
                    continue
                if any(f[2] is flt for j in jobs if j[0] == gi and j[1] == pj for f in j[5]):
                    continue
                out[gi][pj] = _device_filter(out[gi][pj], flt.variable, flt.regex, dictionary)
    return out


def _reduced_tables(ds: DeviceStore, g, tables: list, jv: list, needed) -> list:
    """Semi-join reduce a group's scanned tables (columns: #idx + join
    variables) and materialise each pattern's live columns."""
    tabs = [DevTable([_IDX] + [v for v in pat.variables() if v in jv], t) for pat, t in zip(g.patterns, tables)]
    n_bits = ds.id_bound()
    for v in jv:
        ids = [j for j, t in enumerate(tabs) if v in t.columns]
        if len(ids) < 2:
            continue
        hs = (ctypes.c_void_p * len(ids))(*[tabs[j].t.handle.value for j in ids])
        outs = (ctypes.c_void_p * len(ids))()
        _lib.call("tidq_tables_semijoin", len(ids), hs, _i32([tabs[j].col(v) for j in ids]), n_bits, outs)
        for k, j in enumerate(ids):
            tabs[j] = DevTable(tabs[j].columns, _lib.DeviceTable(ctypes.c_void_p(outs[k])))
    res = []
    for pat, vs, t in zip(g.patterns, g.var_slots, tabs):
        live = _live_columns(pat, needed)
        spec = [t.col(v) if v in t.columns else -1 - vs[v][0] for v in live]
        h = _new_handle("tidq_store_gather_cols", ds.handle, t.t.handle, 0, len(spec), _i32(spec))
        r = DevTable.from_handle(live, h)
        r.reduced = True
        res.append(r)
    return res


def _capacity_hints(ds: DeviceStore, spec: _lib.ScanSpec, keys: list) -> None:
    """Exact/upper-bound output sizes from the store's predicate histogram
    for streams whose key binds the predicate (lets the scan skip its
    mid-pass host sync).  Streams without a bound predicate get no hint."""
    hist = ds.predicate_counts()
    if hist is None:
        return
    for s in range(spec.n_streams):
        st = spec.streams[s]
        hint = 0
        for q, (ks, kp, ko) in enumerate(keys):
            if not (st.select >> q) & 1:
                continue
            if kp == 0:
                hint = 0
                break
            hint += int(hist[kp]) if kp < len(hist) else 0
        else:
            st.capacity_hint = max(hint, 1)


def _units(store, chunk_triples):
    items, host = _as_stores(store, chunk_triples)
    for it in items:
        yield it, host


def scan_patterns(groups: Sequence, store, workers: int = 1, chunk_triples: int | None = None):
    """Matched (n, 3) uint32 rows per group and pattern (query_ops.py:263-295),
    from ONE device pass over all groups' keys per chunk."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    ctx = _lib.context()
    jobs = [(gi, pj, key) for gi, g in enumerate(groups) if g.satisfiable for pj, key in enumerate(g.keys)]
    parts: dict = {}
    for unit, host in _units(store, chunk_triples):
        ds = DeviceStore.upload(unit) if host else unit
        try:
            for lo in range(0, len(jobs), _lib.MAX_STREAMS):
                batch = jobs[lo: lo + _lib.MAX_STREAMS]
                keys: list = []
                spec = _lib.ScanSpec()
                spec.n_streams = len(batch)
                for s, (gi, pj, key) in enumerate(batch):
                    k = (int(key.subj), int(key.pred), int(key.obj))
                    if k not in keys:
                        keys.append(k)
                    st = spec.streams[s]
                    st.select = 1 << keys.index(k)
                    st.n_out = 3
                    st.out[0], st.out[1], st.out[2] = _lib.OUT_S, _lib.OUT_P, _lib.OUT_O
                spec.n_keys = len(keys)
                for q, k in enumerate(keys):
                    spec.keys[q][:] = k
                for (gi, pj, _), t in zip(batch, _lib.run_scan(ds.handle, spec)):
                    try:
                        if t.n_rows:
                            parts.setdefault((gi, pj), []).append(
                                np.stack([t.column(0), t.column(1), t.column(2)], axis=1))
                    finally:
                        t.free()
        finally:
            if host:
                ds.free()
    del ctx
    return [[np.concatenate(parts[(gi, pj)]) if (gi, pj) in parts else np.empty((0, 3), ID_DTYPE)
             for pj in range(len(g.keys))] for gi, g in enumerate(groups)]


# ----------------------------------------------------------------------------- joins


def merge_join(left, right) -> np.ndarray:
    """All (l, r) index pairs with equal keys, ordered by key, then l, then r
    (query_ops.py:144-177), computed by the device sort-merge join."""
    lk = np.ascontiguousarray(left.key if isinstance(left, BindingRelation) else np.asarray(left),
                              dtype=np.uint32)
    rk = np.ascontiguousarray(right.key if isinstance(right, BindingRelation) else np.asarray(right),
                              dtype=np.uint32)
    if len(lk) == 0 or len(rk) == 0:
        return np.empty((0, 2), dtype=np.int64)
    ctx = _lib.context()
    t = _lib.DeviceTable(_new_handle("tidq_merge_join_pairs", ctx.handle, _lib.ptr(lk), len(lk),
                                     _lib.ptr(rk), len(rk)))
    try:
        if t.n_rows == 0:
            return np.empty((0, 2), dtype=np.int64)
        return np.stack([t.column(0), t.column(1)], axis=1)
    finally:
        t.free()


def _group_result(store, compiled, cg, tables: list[DevTable], row_cap, key_bound: int = 0) -> DevTable:
    """The group's join chain, then its deferred variables gathered."""
    t = _join_chain(cg, tables, row_cap, key_bound)
    if t.columns and any(c.startswith(_DEF) for c in t.columns):
        t = _materialize(store, cg, t, _needed_variables(compiled, cg))
    return t


def _join_chain(cg, tables: list[DevTable], row_cap, key_bound: int = 0) -> DevTable:
    """Left-deep chain of joins in analyze_relationships order.  ``key_bound``
    (the store's largest ID + 1, when the tables came from one) spares each
    join its max pass over the keys."""
    rels = analyze_relationships(cg.patterns)
    # tables that went through the scan's semi-join reduction skip the join's
    # own key-bitmap pre-filter (a pure optimisation either way)
    algo = JOIN_REDUCED if tables and all(getattr(t, "reduced", False) for t in tables) else 0
    acc = tables[0]
    for rel in rels:
        acc = _dev_join(acc, tables[rel.j], rel.variable, row_cap, algo, key_bound)
    return acc


def pattern_table(pattern, var_slots: dict, rows: np.ndarray) -> BindingTable:
    """Bindings of one pattern's variables from its matched triples
    (query_ops.py:210-229); rows whose repeated-variable slots differ dropped."""
    rows = np.ascontiguousarray(np.asarray(rows, dtype=ID_DTYPE).reshape(-1, 3))
    outs, eq = _pattern_spec(pattern, var_slots)
    cols = pattern.variables()
    if not len(rows):
        return BindingTable(cols, {c: np.empty(0, ID_DTYPE) for c in cols})
    # the rows form a tiny store; the ??? key selects all, the epilogue masks
    spec = _lib.ScanSpec()
    spec.n_keys = 1
    spec.n_streams = 1
    st = spec.streams[0]
    st.select = 1
    st.eq_flags = eq
    st.n_out = len(outs)
    for k, slot in enumerate(outs):
        st.out[k] = slot
    ctx = _lib.context()
    (t,) = _lib.run_scan(ctx.handle, spec, host=(rows.reshape(-1), len(rows), 0))
    return DevTable(cols, t).download()


def join_group(cg, pattern_rows: Sequence[np.ndarray], dictionary, row_cap: int | None = DEFAULT_ROW_CAP) -> BindingTable:
    """Filter and join one group's pattern results (query_ops.py:298-342)."""
    ctx = _lib.context()
    tables = []
    for pat, vs, rows in zip(cg.patterns, cg.var_slots, pattern_rows):
        bt = pattern_table(pat, vs, rows)
        tables.append(DevTable.upload(bt.columns, bt.data, ctx))
    for flt in cg.filters:
        tables = [_device_filter(t, flt.variable, flt.regex, dictionary) if flt.variable in t.columns else t
                  for t in tables]
    return _join_chain(cg, tables, row_cap).download()


def evaluate_group(group, store, dictionary, workers: int = 1, chunk_triples: int | None = None,
                   row_cap: int | None = DEFAULT_ROW_CAP) -> BindingTable:
    """Search, filter and join one group against a store (query_ops.py:345-356)."""
    cg = group if hasattr(group, "keys") and hasattr(group, "satisfiable") else compile_group(group, dictionary)
    if workers < 1:
        raise ValueError("workers must be >= 1")
    resident = isinstance(store, DeviceStore)
    tables = _scan_device(_units(store, chunk_triples), [cg], dictionary, fuse_filters=True,
                          semijoin=row_cap is None, defer=resident)[0]
    return _group_result(store, None, cg, tables, row_cap, store.id_bound() if resident else 0).download()


def _union_device(tables: list[DevTable]) -> DevTable:
    cols: list = []
    for t in tables:
        for c in t.columns:
            if c not in cols:
                cols.append(c)
    if all(t.columns == cols for t in tables) and all(t.n_rows == 0 for t in tables[1:]):
        return tables[0]  # (a TIDQ_SCAN_CONCAT scan already wrote the union)
    return _dev_concat(_lib.context(), tables, cols)


def evaluate_union(tables: Sequence[BindingTable]) -> BindingTable:
    """Concatenate branch tables over the union of their columns; absent
    columns are UNBOUND (query_ops.py:359-376)."""
    ctx = _lib.context()
    dts = [DevTable.upload(t.columns, t.data, ctx) for t in tables]
    if not dts:
        return BindingTable([], {})
    return _union_device(dts).download()


def _project_distinct_device(t: DevTable, projection, distinct: bool, key_bound: int = 0) -> DevTable:
    cols = list(projection) if projection is not None else list(t.columns)
    missing = [c for c in cols if c not in t.columns]
    if missing:
        raise KeyError(f"projection names unbound variables: {missing}")
    if not distinct or t.n_rows == 0:
        return _dev_project(t, cols) if cols else DevTable([], None)
    return _dev_distinct(t, cols, key_bound)


def project_distinct(table: BindingTable, projection, distinct: bool) -> BindingTable:
    """Projection, then optional DISTINCT keeping first occurrences
    (query_ops.py:379-399)."""
    cols = list(projection) if projection is not None else list(table.columns)
    missing = [c for c in cols if c not in table.data]
    if missing:
        raise KeyError(f"projection names unbound variables: {missing}")
    out = BindingTable(cols, {c: table.data[c] for c in cols})
    if not distinct or out.n_rows == 0:
        return out
    return _dev_distinct(DevTable.upload(cols, out.data), cols).download()


def decode_table(table: BindingTable, dictionary) -> str:
    """TSV rendering (query_ops.py:402-423): a header of ?-prefixed variable
    names, then one line per row of verbatim terms, empty cells for UNBOUND.

    Every distinct ID is decoded once; the text is then assembled with a
    single join over a (rows x 2*columns) object grid of cells and
    separators instead of one join per row."""
    header = "\t".join("?" + c for c in table.columns) + "\n"
    n, k = table.n_rows, len(table.columns)
    if not n or not k:
        return header
    grid = np.empty((n, 2 * k), dtype=object)
    grid[:, 1::2] = "\t"
    grid[:, -1] = "\n"
    for j, c in enumerate(table.columns):
        ids, where = np.unique(np.asarray(table.data[c]), return_inverse=True)
        text = np.array([dictionary.decode_lexical(int(i)) if i != UNBOUND else "" for i in ids.tolist()],
                        dtype=object)
        grid[:, 2 * j] = text[where.reshape(-1)]
    return header + "".join(grid.ravel().tolist())


@dataclass
class QueryTimings:
    search: float = 0.0
    join: float = 0.0


def _concat_union(compiled, store) -> bool:
    """A UNION whose branches are single patterns with the same live
    columns, no FILTER, on one resident store: scanned into one table."""
    groups = compiled.groups
    if not isinstance(store, DeviceStore) or not 2 <= len(groups) <= _lib.MAX_STREAMS:
        return False
    if any(not g.satisfiable or len(g.patterns) != 1 or g.filters for g in groups):
        return False
    cols = [_live_columns(g.patterns[0], _needed_variables(compiled, g)) for g in groups]
    return all(c == cols[0] for c in cols)


def evaluate_query_device(compiled, store, dictionary, workers: int = 1, chunk_triples=None,
                          row_cap: int | None = DEFAULT_ROW_CAP, timings: QueryTimings | None = None) -> DevTable:
    """evaluate_query keeping the result on the device (a DevTable)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    t0 = perf_counter()
    resident = isinstance(store, DeviceStore)
    per_group = _scan_device(_units(store, chunk_triples), compiled.groups, dictionary, fuse_filters=True,
                             compiled=compiled, concat=_concat_union(compiled, store),
                             semijoin=row_cap is None, defer=resident)
    t1 = perf_counter()
    bound = store.id_bound() if resident else 0
    branches = [_group_result(store, compiled, cg, tables, row_cap, bound)
                for cg, tables in zip(compiled.groups, per_group)]
    union = _union_device(branches)
    result = _project_distinct_device(union, compiled.projection, compiled.distinct, bound)
    t2 = perf_counter()
    if timings is not None:
        timings.search = t1 - t0
        timings.join = t2 - t1
    return result


def evaluate_query(compiled, store, dictionary, workers: int = 1, chunk_triples: int | None = None,
                   row_cap: int | None = DEFAULT_ROW_CAP, timings: QueryTimings | None = None) -> BindingTable:
    """Full pipeline for a compiled query: scan, join, union, project
    (query_ops.py:432-455); the result is downloaded as a BindingTable."""
    t0 = perf_counter()
    res = evaluate_query_device(compiled, store, dictionary, workers, chunk_triples, row_cap, timings)
    out = res.download()
    if timings is not None:
        timings.join += perf_counter() - t0 - timings.search - timings.join
    return out
