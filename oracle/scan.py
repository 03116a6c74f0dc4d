"""Oracle scan — restates reference kernel.py:139-227 and query_ops.py:263-295.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Structure follows the
reference CPU path: the triple range is cut into 65,536-triple tiles handed
round-robin to W threads (kernel.py:99-132); each tile evaluates every key
slot by slot with strided compares on the AoS rows (kernel.py:205-222); one
sequential ``nonzero`` compacts (kernel.py:177-179, 226-227).
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

TILE = 1 << 16
MAX_KEYS = 32


def _ids(key) -> tuple[int, int, int]:
    return int(key.subj), int(key.pred), int(key.obj)


def _mask(key) -> int:
    s, p, o = _ids(key)
    return (4 if s else 0) | (2 if p else 0) | (1 if o else 0)


def _tiles(n: int, workers: int):
    """kernel.py:99-107: tile t goes to worker t % W."""
    per = [[] for _ in range(workers)]
    for t, lo in enumerate(range(0, n, TILE)):
        per[t % workers].append((lo, min(n, lo + TILE)))
    return per


def _parallel(fn, workers: int) -> None:
    if workers == 1:
        fn(0)
        return
    with ThreadPoolExecutor(max_workers=workers) as ex:
        list(ex.map(fn, range(workers)))


def search_chunk(chunk, key, workers: int = 1):
    """kernel.py:148-179 -> (int64 global indices, uint8 answer codes)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    rows = np.asarray(chunk.data).reshape(-1, 3)
    n = len(rows)
    codes = np.zeros(n, dtype=np.uint8)
    k = np.array(_ids(key), dtype=np.uint32)
    spans = _tiles(n, workers)

    def run(w):
        for lo, hi in spans[w]:
            t = rows[lo:hi]
            codes[lo:hi] = ((t[:, 0] == k[0]).astype(np.uint8) << 2) | (
                (t[:, 1] == k[1]).astype(np.uint8) << 1) | (t[:, 2] == k[2]).astype(np.uint8)

    _parallel(run, workers)
    m = _mask(key)
    hit = np.flatnonzero((codes & m) == m)
    return hit.astype(np.int64) + int(chunk.base_index), codes[hit]


def search_multi(chunk, keys, workers: int = 1):
    """kernel.py:182-227 -> (int64 global indices, uint32 mark sets)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    keys = list(keys)
    if not 1 <= len(keys) <= MAX_KEYS:
        raise ValueError(f"{len(keys)} keys; supported range is 1..{MAX_KEYS}")
    rows = np.asarray(chunk.data).reshape(-1, 3)
    n = len(rows)
    marks = np.zeros(n, dtype=np.uint32)
    key_ids = [_ids(k) for k in keys]
    spans = _tiles(n, workers)

    def run(w):
        for lo, hi in spans[w]:
            t = rows[lo:hi]
            acc = np.zeros(hi - lo, dtype=np.uint32)
            for q, ids in enumerate(key_ids):
                bit = np.uint32(1 << q)
                ok = None
                for slot in range(3):
                    if ids[slot]:
                        eq = t[:, slot] == ids[slot]
                        ok = eq if ok is None else ok & eq
                if ok is None:  # ??? key marks every triple (kernel.py:210-212)
                    acc |= bit
                else:
                    acc |= ok.astype(np.uint32) << np.uint32(q)
            marks[lo:hi] = acc

    _parallel(run, workers)
    hit = np.flatnonzero(marks)
    return hit.astype(np.int64) + int(chunk.base_index), marks[hit]


def _as_chunks(store):
    if hasattr(store, "data") and hasattr(store, "base_index"):
        return [store]
    return list(store)


def scan_patterns(groups, store, workers: int = 1):
    """query_ops.py:263-295: per group, per pattern, matched (n,3) uint32 rows
    in ascending triple order; unsatisfiable groups yield empty lists."""
    acc = [[[] for _ in g.keys] for g in groups]
    for chunk in _as_chunks(store):
        rows_all = np.asarray(chunk.data).reshape(-1, 3)
        for gi, g in enumerate(groups):
            if not g.satisfiable:
                continue
            idx, marks = search_multi(chunk, g.keys, workers)
            if not len(idx):
                continue
            rows = rows_all[idx - int(chunk.base_index)]
            for q in range(len(g.keys)):
                sel = ((marks >> np.uint32(q)) & np.uint32(1)).astype(bool)
                if sel.any():
                    acc[gi][q].append(rows[sel])
    return [[np.concatenate(p) if p else np.empty((0, 3), dtype=np.uint32) for p in g] for g in acc]
