"""Two-stage search pipelines for the six two-pattern RDFS rules — drop-in for
reference ``tripleid.entailment`` (entailment.py:1-255), searches on the B200.

    R2   s p o,  p rdfs:domain D          =>  s rdf:type D
    R3   s p o,  p rdfs:range R           =>  o rdf:type R
    R7   s p o,  p rdfs:subPropertyOf q   =>  s q o
    R5   p rdfs:subPropertyOf q,  q rdfs:subPropertyOf r  =>  p rdfs:subPropertyOf r
    R9   s rdf:type x,  x rdfs:subClassOf y    =>  s rdf:type y
    R11  x rdfs:subClassOf y,  y rdfs:subClassOf z  =>  x rdfs:subClassOf z

Same rule table, RuleRun, report_counts and run_rule signature and results.
What changes is stage 2.  The reference issues one search key per distinct
link value, 32 keys per full pass over the store (entailment.py:130-156:
ceil(links/32) passes — 148 passes for the paper's 4,716 links,
PAPER.md:1272).  Here stage 2 is ONE device scan whatever the number of
links: the link values become a bitmap over term IDs, tested as a scan
epilogue predicate —

  * rules whose stage-2 key is (link, pred2, 0) (R5, R9, R11): key
    (0, pred2, 0) with the subject tested against the link bitmap;
  * rules whose stage-2 key is (0, link, 0) (R2, R3, R7): the all-triples key
    with the predicate tested against the link bitmap.

The match set, the ascending index order, the hash tables, the conclusion set
and the report counts equal the reference's (tests/test_gpu_entail.py against
golden vectors from the reference run_rule).  ``res2`` — the reference's
count of accepted (triple, key) pairs — is the number of stage-2 triples with
distinct keys, and the multiplicity-weighted count when
``deduplicate=False`` sends repeated link values as repeated keys.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum
from time import perf_counter
from typing import Callable

import numpy as np

from . import _lib
from .query_ops import _DeviceBitmap, _as_stores
from .store import DeviceStore

RDF_TYPE = "<http://www.w3.org/1999/02/22-rdf-syntax-ns#type>"
RDFS_DOMAIN = "<http://www.w3.org/2000/01/rdf-schema#domain>"
RDFS_RANGE = "<http://www.w3.org/2000/01/rdf-schema#range>"
RDFS_SUBPROPERTY = "<http://www.w3.org/2000/01/rdf-schema#subPropertyOf>"
RDFS_SUBCLASS = "<http://www.w3.org/2000/01/rdf-schema#subClassOf>"

SUBJ, PRED, OBJ = 0, 1, 2


class Role(IntEnum):
    """dictionary.py:30-33 (the role passed to Dictionary.encode_lexical)."""

    SUBJECT = 0
    PREDICATE = 1
    OBJECT = 2


@dataclass(frozen=True)
class EntailmentRule:
    """One two-pattern rule in pipeline form (entailment.py:46-67)."""

    rule_id: int
    stage1_pred: str
    link_slot: int
    partner_slot: int
    stage2_pred: str | None
    value_slots: tuple[int, ...]
    conclusion_pred: str
    conclude: Callable[[int, tuple[int, ...], int], tuple[int, int, int]]


RULES: dict[int, EntailmentRule] = {  # entailment.py:70-94
    2: EntailmentRule(2, RDFS_DOMAIN, SUBJ, OBJ, None, (SUBJ,), RDF_TYPE,
                      lambda d, v, pred: (v[0], pred, d)),
    3: EntailmentRule(3, RDFS_RANGE, SUBJ, OBJ, None, (OBJ,), RDF_TYPE,
                      lambda r, v, pred: (v[0], pred, r)),
    7: EntailmentRule(7, RDFS_SUBPROPERTY, SUBJ, OBJ, None, (SUBJ, OBJ), "",
                      lambda q, v, pred: (v[0], q, v[1])),
    5: EntailmentRule(5, RDFS_SUBPROPERTY, OBJ, SUBJ, RDFS_SUBPROPERTY, (OBJ,), RDFS_SUBPROPERTY,
                      lambda p, v, pred: (p, pred, v[0])),
    9: EntailmentRule(9, RDF_TYPE, OBJ, SUBJ, RDFS_SUBCLASS, (OBJ,), RDF_TYPE,
                      lambda s, v, pred: (s, pred, v[0])),
    11: EntailmentRule(11, RDFS_SUBCLASS, OBJ, SUBJ, RDFS_SUBCLASS, (OBJ,), RDFS_SUBCLASS,
                       lambda x, v, pred: (x, pred, v[0])),
}


@dataclass
class RuleRun:
    """Everything one rule application produced (entailment.py:96-114)."""

    rule_id: int
    stage1_indices: np.ndarray
    stage1_table: dict[int, set[int]]
    stage2_indices: np.ndarray
    stage2_table: dict[int, set]
    conclusions: set[tuple[int, int, int]]
    res1: int = 0
    res2: int = 0

    @property
    def dist1(self) -> int:
        return len(self.stage1_table)

    @property
    def dist2(self) -> int:
        return sum(len(v) for v in self.stage2_table.values())


def report_counts(run: RuleRun) -> tuple[int, int, int, int, int]:
    """(res1, dist1, res2, dist2, all) (entailment.py:117-119)."""
    return (run.res1, run.dist1, run.res2, run.dist2, len(run.conclusions))


# ---- device searches --------------------------------------------------------------


def _id_bitmap(ids: np.ndarray) -> tuple[np.ndarray, int]:
    ids = np.asarray(ids, dtype=np.uint64)
    n_bits = int(ids.max()) + 1 if ids.size else 1
    words = np.zeros((n_bits + 31) // 32, dtype=np.uint32)
    np.bitwise_or.at(words, (ids >> np.uint64(5)).astype(np.int64),
                     (np.uint32(1) << (ids & np.uint64(31)).astype(np.uint32)))
    return words, n_bits


def _search(units, key: tuple[int, int, int], set_slot: int | None = None, set_ids=None):
    """(ascending global indices int64, rows (n, 3) uint32) of the triples
    matching ``key`` (and, with ``set_slot``, whose value in that slot is one
    of ``set_ids``): one device scan per store unit."""
    ctx = _lib.context()
    bitmap = None
    if set_slot is not None:
        words, n_bits = _id_bitmap(set_ids)
        bitmap = _DeviceBitmap(ctx, words, n_bits)
    idx_parts, row_parts = [], []
    for unit, host in units:
        spec = _lib.ScanSpec()
        spec.n_keys = 1
        spec.keys[0][:] = key
        spec.n_streams = 1
        st = spec.streams[0]
        st.select = 1
        st.n_out = 4
        st.out[0] = _lib.OUT_INDEX
        st.out[1], st.out[2], st.out[3] = _lib.OUT_S, _lib.OUT_P, _lib.OUT_O
        if bitmap is not None:
            st.n_filters = 1
            st.filter_slot[0] = set_slot
            st.filter[0] = bitmap.handle.value
        if host:
            data = np.ascontiguousarray(unit.data, dtype=np.uint32).reshape(-1)
            (t,) = _lib.run_scan(ctx.handle, spec, host=(data, data.size // 3, int(unit.base_index)))
        else:
            (t,) = _lib.run_scan(unit.handle, spec)
        try:
            if t.n_rows:
                idx_parts.append(t.column(0))
                row_parts.append(np.stack([t.column(1), t.column(2), t.column(3)], axis=1))
        finally:
            t.free()
    if not idx_parts:
        return np.empty(0, dtype=np.int64), np.empty((0, 3), dtype=np.uint32)
    return np.concatenate(idx_parts), np.concatenate(row_parts)


def _group(link: np.ndarray, values: np.ndarray) -> dict:
    """{link: set(value or value tuple)} from parallel arrays (one value
    column -> ints, several -> tuples)."""
    if not len(link):
        return {}
    cols = [link.astype(np.int64)] + [values[:, j].astype(np.int64) for j in range(values.shape[1])]
    uniq = np.unique(np.stack(cols, axis=1), axis=0)
    heads = np.flatnonzero(np.r_[True, uniq[1:, 0] != uniq[:-1, 0]])
    bounds = np.r_[heads, len(uniq)]
    out = {}
    single = values.shape[1] == 1
    for a, b in zip(bounds[:-1].tolist(), bounds[1:].tolist()):
        vals = uniq[a:b, 1:]
        out[int(uniq[a, 0])] = set(vals[:, 0].tolist()) if single else set(map(tuple, vals.tolist()))
    return out


def _conclusions(rule: EntailmentRule, table1: dict, table2: dict, dictionary) -> set:
    """Join of the two tables on the link (entailment.py:236-253), with the
    conclusion predicate encoded on first use exactly as the reference does."""
    shared = [link for link in table2 if table1.get(link)]
    if not shared:
        return set()
    pred = 0
    if rule.conclusion_pred:
        pred = dictionary.encode_lexical(rule.conclusion_pred, Role.PREDICATE)
    out = set()
    for link in shared:
        partners = table1[link]
        for value in table2[link]:
            v = value if isinstance(value, tuple) else (value,)
            for partner in partners:
                out.add(rule.conclude(partner, v, pred))
    return out


def run_rule(rule, store, dictionary, workers: int = 1, chunk_triples: int | None = None,
             deduplicate: bool = True, *, timings: dict | None = None) -> RuleRun:
    """Apply one rule over a store; single application, no fixpoint
    (entailment.py:175-255).  ``store``: DeviceStore (resident), TripleChunk,
    list of chunks, or a .tid path.  ``timings`` (optional, not in the
    reference) receives the seconds spent in the two device searches
    ("search") and in building the Python tables and conclusions ("tables")."""
    t_search = t_tables = 0.0
    if isinstance(rule, int):
        rule = RULES[rule]
    empty = RuleRun(rule.rule_id, np.empty(0, dtype=np.int64), {}, np.empty(0, dtype=np.int64), {}, set())
    pred1 = dictionary.lookup(rule.stage1_pred)
    if pred1 is None:
        return empty
    pred2 = None
    if rule.stage2_pred is not None:
        pred2 = dictionary.lookup(rule.stage2_pred)
        if pred2 is None:
            return empty
    if workers < 1:  # kernel.py:161-162 (raised by the first search)
        raise ValueError("workers must be >= 1")
    items, host = _as_stores(store, chunk_triples)
    units = [(it, host and not isinstance(it, DeviceStore)) for it in items]

    t0 = perf_counter()
    idx1, rows1 = _search(units, (0, int(pred1), 0))
    t1 = perf_counter()
    res1 = len(idx1)  # one key: accepted pairs = matched triples
    table1 = _group(rows1[:, rule.link_slot], rows1[:, [rule.partner_slot]])
    t_search += t1 - t0
    t_tables += perf_counter() - t1
    if timings is not None:
        timings.update(search=t_search, tables=t_tables)
    if not table1:
        empty.res1 = res1
        return empty

    link_col2 = PRED if pred2 is None else SUBJ
    links = np.fromiter(table1.keys(), dtype=np.uint64, count=len(table1))
    t0 = perf_counter()
    if pred2 is None:  # keys (0, link, 0): any triple whose predicate is a link
        idx2, rows2 = _search(units, (0, 0, 0), PRED, links)
    else:  # keys (link, pred2, 0)
        idx2, rows2 = _search(units, (0, int(pred2), 0), SUBJ, links)
    t1 = perf_counter()
    if deduplicate:
        res2 = len(idx2)
    else:  # every stage-1 row sends its link as a key: pairs = link multiplicities
        lv, lc = np.unique(rows1[:, rule.link_slot], return_counts=True)
        res2 = int(lc[np.searchsorted(lv, rows2[:, link_col2])].sum()) if len(idx2) else 0
    table2 = _group(rows2[:, link_col2], rows2[:, list(rule.value_slots)])
    conclusions = _conclusions(rule, table1, table2, dictionary)
    if timings is not None:
        timings.update(search=t_search + t1 - t0, tables=t_tables + perf_counter() - t1)
    return RuleRun(rule.rule_id, idx1, table1, idx2, table2, conclusions, res1, res2)
