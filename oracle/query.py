"""Oracle query operators — restates reference query_ops.py:63-455.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Semantics kept exactly:
bag semantics everywhere, DISTINCT the only dedup (first occurrence kept),
UNBOUND = 0 in UNION, repeated-variable rows dropped, FILTER applied to every
pattern table binding the variable before any join, left-deep joins in the
order of ``analyze_relationships``, ``ResourceLimit`` when the pair count of a
join exceeds ``row_cap``.  Row order follows the reference too (merge_join
orders pairs by key, then left row, then right row).
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field

import numpy as np

from . import scan as oscan

UNBOUND = 0
SLOT_LETTERS = ("S", "P", "O")


class DisconnectedPatterns(ValueError):
    pass


class ResourceLimit(RuntimeError):
    pass


@dataclass
class Table:
    """query_ops.py:180-207 BindingTable: one uint32 column per variable."""

    columns: list
    data: dict = field(default_factory=dict)

    @property
    def n_rows(self) -> int:
        return len(self.data[self.columns[0]]) if self.columns else 0

    def take(self, idx) -> "Table":
        return Table(list(self.columns), {c: self.data[c][idx] for c in self.columns})

    def rows(self) -> np.ndarray:
        if not self.columns:
            return np.empty((0, 0), dtype=np.uint32)
        return np.stack([np.asarray(self.data[c], dtype=np.uint32) for c in self.columns], axis=1)


def _is_var(slot) -> bool:
    return hasattr(slot, "name")


def pattern_table(pattern, var_slots, rows) -> Table:
    """query_ops.py:210-229: first slot per variable; rows whose repeated
    variable slots disagree are dropped."""
    rows = np.asarray(rows, dtype=np.uint32).reshape(-1, 3)
    keep = np.ones(len(rows), dtype=bool)
    for slots in var_slots.values():
        first = slots[0]
        for other in slots[1:]:
            keep &= rows[:, first] == rows[:, other]
    rows = rows[keep]
    names = pattern.variables()
    return Table(names, {v: rows[:, var_slots[v][0]].copy() for v in names})


def str_form(lexical: str) -> str:
    """query_ops.py:232-238."""
    if lexical.startswith("<"):
        return lexical[1:-1]
    if lexical.startswith('"'):
        return lexical[1:lexical.rfind('"')]
    return lexical


def accepted_ids(ids, regex: str, dictionary) -> np.ndarray:
    """IDs among ``ids`` whose str() form matches ``regex`` (re.search)."""
    rx = re.compile(regex)
    uniq = np.unique(np.asarray(ids, dtype=np.uint32))
    ok = [u for u in uniq.tolist() if rx.search(str_form(dictionary.decode_lexical(u)))]
    return np.array(ok, dtype=np.uint32)


def apply_filter(table: Table, variable: str, regex: str, dictionary) -> Table:
    """query_ops.py:241-252."""
    col = table.data[variable]
    keep = np.isin(col, accepted_ids(col, regex, dictionary))
    return table.take(np.flatnonzero(keep))


def analyze_relationships(patterns):
    """query_ops.py:63-91: pattern j links to the closest earlier pattern
    sharing a variable; the join variable is the shared one with the smallest
    first slot in pattern i.  Returns (i, j, type, var) tuples."""
    if len(patterns) < 2:
        return []
    maps = [p.var_slots() for p in patterns]
    rels = []
    for j in range(1, len(patterns)):
        found = None
        for i in range(j - 1, -1, -1):
            common = [v for v in maps[i] if v in maps[j]]
            if common:
                var = min(common, key=lambda v: maps[i][v][0])
                found = (i, j, SLOT_LETTERS[maps[i][var][0]] + SLOT_LETTERS[maps[j][var][0]], var)
                break
        if found is None:
            raise DisconnectedPatterns(f"pattern {j} shares no variable with any earlier pattern")
        rels.append(found)
    return rels


def build_relation(rows, pattern, join_slot: str):
    """query_ops.py:121-136: (key, {slot letter: column}) of the two non-key
    slots; the join slot must be a variable slot (ValueError otherwise)."""
    idx = SLOT_LETTERS.index(join_slot)
    slot = pattern.slots[idx]
    if not pattern.var_slots().get(slot.name if _is_var(slot) else None):
        raise ValueError(f"join slot {join_slot} is not a variable of the pattern")
    rows = np.asarray(rows).reshape(-1, 3)
    return rows[:, idx].copy(), {SLOT_LETTERS[k]: rows[:, k].copy() for k in range(3) if k != idx}


def prepare_for_join(key, values):
    """query_ops.py:110-118: stable sort by key, values permuted alike."""
    order = np.argsort(key, kind="stable")
    return key[order], {k: v[order] for k, v in values.items()}


def merge_join(left_keys, right_keys) -> np.ndarray:
    """query_ops.py:144-177: all (l, r) with equal keys, ordered by
    (key asc, l asc, r asc); equal-key runs give their cross product."""
    lk = np.asarray(left_keys)
    rk = np.asarray(right_keys)
    if len(lk) == 0 or len(rk) == 0:
        return np.empty((0, 2), dtype=np.int64)
    lo = np.argsort(lk, kind="stable").astype(np.int64)
    ro = np.argsort(rk, kind="stable").astype(np.int64)
    ls, rs = lk[lo], rk[ro]
    start = np.searchsorted(rs, ls, "left")
    stop = np.searchsorted(rs, ls, "right")
    cnt = stop - start
    total = int(cnt.sum())
    if total == 0:
        return np.empty((0, 2), dtype=np.int64)
    left = np.repeat(lo, cnt)
    # right positions: for each left row, the run start..stop of the sorted right
    offs = np.repeat(np.cumsum(cnt) - cnt, cnt)
    pos = np.arange(total, dtype=np.int64) - offs + np.repeat(start, cnt)
    return np.stack([left, ro[pos]], axis=1)


def merge_join_loop(left_keys, right_keys) -> np.ndarray:
    """query_ops.py:144-177 step for step — stable argsorts, intersect1d,
    searchsorted run bounds, then the Python loop over common keys with
    repeat/tile.  Same output as merge_join; used where the reference's CPU
    COST is what is measured (bench.py's CPU baselines), not for parity."""
    lk = np.asarray(left_keys)
    rk = np.asarray(right_keys)
    if len(lk) == 0 or len(rk) == 0:
        return np.empty((0, 2), dtype=np.int64)
    lo = np.argsort(lk, kind="stable").astype(np.int64)
    ro = np.argsort(rk, kind="stable").astype(np.int64)
    ls, rs = lk[lo], rk[ro]
    common = np.intersect1d(ls, rs)
    if len(common) == 0:
        return np.empty((0, 2), dtype=np.int64)
    l_start = np.searchsorted(ls, common, "left")
    l_end = np.searchsorted(ls, common, "right")
    r_start = np.searchsorted(rs, common, "left")
    r_end = np.searchsorted(rs, common, "right")
    l_parts, r_parts = [], []
    for k in range(len(common)):
        li = lo[l_start[k]: l_end[k]]
        ri = ro[r_start[k]: r_end[k]]
        l_parts.append(np.repeat(li, len(ri)))
        r_parts.append(np.tile(ri, len(li)))
    return np.stack([np.concatenate(l_parts), np.concatenate(r_parts)], axis=1)


def join_group(cg, pattern_rows, dictionary, row_cap=10_000_000, faithful: bool = False) -> Table:
    """query_ops.py:298-342."""
    tables = [pattern_table(p, vs, r) for p, vs, r in zip(cg.patterns, cg.var_slots, pattern_rows)]
    for flt in cg.filters:
        tables = [apply_filter(t, flt.variable, flt.regex, dictionary) if flt.variable in t.data else t
                  for t in tables]
    acc = tables[0]
    for i, j, _typ, var in analyze_relationships(cg.patterns):
        right = tables[j]
        pairs = (merge_join_loop if faithful else merge_join)(acc.data[var], right.data[var])
        if row_cap is not None and len(pairs) > row_cap:
            raise ResourceLimit(f"join produced {len(pairs)} rows, cap is {row_cap}")
        li, ri = pairs[:, 0], pairs[:, 1]
        cols = list(acc.columns)
        data = {c: acc.data[c][li] for c in acc.columns}
        keep = None
        for c in right.columns:
            if c == var:
                continue
            rc = right.data[c][ri]
            if c in data:
                eq = data[c] == rc
                keep = eq if keep is None else keep & eq
            else:
                cols.append(c)
                data[c] = rc
        acc = Table(cols, data)
        if keep is not None:
            acc = acc.take(np.flatnonzero(keep))
    return acc


def evaluate_union(tables) -> Table:
    """query_ops.py:359-376: concat over the first-seen union of columns,
    absent columns = UNBOUND (0); no dedup."""
    cols: list = []
    for t in tables:
        for c in t.columns:
            if c not in cols:
                cols.append(c)
    data = {}
    for c in cols:
        parts = [t.data[c] if c in t.data else np.zeros(t.n_rows, dtype=np.uint32) for t in tables]
        data[c] = np.concatenate(parts).astype(np.uint32) if parts else np.empty(0, np.uint32)
    return Table(cols, data)


def project_distinct(table: Table, projection, distinct: bool, faithful: bool = False) -> Table:
    """query_ops.py:379-399: projection (unknown -> KeyError), DISTINCT keeps
    the first occurrence of each row, in first-occurrence order."""
    cols = list(projection) if projection is not None else list(table.columns)
    missing = [c for c in cols if c not in table.data]
    if missing:
        raise KeyError(f"projection names unbound variables: {missing}")
    out = Table(cols, {c: table.data[c] for c in cols})
    if not distinct or out.n_rows == 0:
        return out
    if faithful:  # query_ops.py:393-398: a Python set of row tuples
        seen: set = set()
        keep: list = []
        for i, row in enumerate(tuple(int(x) for x in r) for r in out.rows()):
            if row not in seen:
                seen.add(row)
                keep.append(i)
        return out.take(np.array(keep, dtype=np.int64))
    if len(cols) <= 2:  # one packed uint64 per row: same first occurrences, ~10x faster at 10^8 rows
        key = np.asarray(out.data[cols[0]], dtype=np.uint64)
        if len(cols) == 2:
            key = (key << np.uint64(32)) | np.asarray(out.data[cols[1]], dtype=np.uint64)
        _, first = np.unique(key, return_index=True)
    else:
        _, first = np.unique(out.rows(), axis=0, return_index=True)
    return out.take(np.sort(first))


def evaluate_group(cg, store, dictionary, workers: int = 1, row_cap=10_000_000) -> Table:
    """query_ops.py:345-356 for a compiled group: scan, then join_group."""
    rows = oscan.scan_patterns([cg], store, workers)[0]
    return join_group(cg, rows, dictionary, row_cap)


def evaluate_query(compiled, store, dictionary, workers: int = 1, row_cap=10_000_000,
                   faithful: bool = False) -> Table:
    """query_ops.py:432-455 (scan -> join per group -> union -> project).
    ``faithful``: the reference's own per-key join loop and per-row DISTINCT
    set (its CPU cost, for baselines); the default vectorized forms give the
    same rows faster (parity tests)."""
    per_group = oscan.scan_patterns(compiled.groups, store, workers)
    branches = [join_group(cg, rows, dictionary, row_cap, faithful) for cg, rows in zip(compiled.groups, per_group)]
    return project_distinct(evaluate_union(branches), compiled.projection, compiled.distinct, faithful)
