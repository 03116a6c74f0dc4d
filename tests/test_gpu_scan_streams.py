"""GPU: the scan's stream outputs (mark -> super_offsets -> emit) are
oracle-exact on multi-tile stores, for every bound-column count, single and
multi key, 1..4 streams, partial last tiles and base offsets; selectivity
extremes; capacity hints that are exact, too small or too large."""

import numpy as np
import pytest

from oracle import scan as osc
from paper_1807_01409_b200 import _lib
from paper_1807_01409_b200.kernel import PatternKey
from paper_1807_01409_b200.store import DeviceStore, TripleChunk

pytestmark = pytest.mark.gpu


def run(ds, keys, streams):
    """streams: list of (select, [out kinds])"""
    spec = _lib.ScanSpec()
    spec.n_keys = len(keys)
    for q, k in enumerate(keys):
        spec.keys[q][:] = k
    spec.n_streams = len(streams)
    for s, (sel, outs) in enumerate(streams):
        st = spec.streams[s]
        st.select = sel
        st.n_out = len(outs)
        for i, o in enumerate(outs):
            st.out[i] = o
    tables = _lib.run_scan(ds.handle, spec)
    out = [[t.column(i) for i in range(t.n_cols)] for t in tables]
    for t in tables:
        t.free()
    return out


def expected(rows, base, keys, streams):
    ch = TripleChunk(rows.reshape(-1), base)
    idx, marks = osc.search_multi(ch, [PatternKey(*k) for k in keys])
    res = []
    for sel, outs in streams:
        m = (marks & np.uint32(sel)) != 0
        ii = idx[m]
        cols = []
        for o in outs:
            if o == _lib.OUT_INDEX:
                cols.append(ii)
            else:
                cols.append(rows[ii - base, o])
        res.append(cols)
    return res


CASES = [
    # (keys, streams)
    ([(0, 3, 0)], [(1, [_lib.OUT_S, _lib.OUT_O])]),
    ([(0, 3, 0)], [(1, [_lib.OUT_S, _lib.OUT_P, _lib.OUT_O, _lib.OUT_INDEX])]),
    ([(7, 0, 0)], [(1, [_lib.OUT_P, _lib.OUT_O])]),
    ([(0, 2, 5)], [(1, [_lib.OUT_S])]),
    ([(4, 2, 5)], [(1, [_lib.OUT_INDEX])]),
    ([(0, 1, 0), (0, 2, 0)], [(1, [_lib.OUT_S, _lib.OUT_O]), (2, [_lib.OUT_O, _lib.OUT_S])]),
    ([(0, 1, 0), (0, 2, 0), (3, 0, 0)], [(1, [_lib.OUT_S]), (2, [_lib.OUT_O]), (4, [_lib.OUT_P, _lib.OUT_O])]),
    ([(0, 1, 0), (0, 2, 0), (0, 3, 0), (0, 4, 0)],
     [(1, [_lib.OUT_S]), (2, [_lib.OUT_S]), (4, [_lib.OUT_S]), (8, [_lib.OUT_S, _lib.OUT_INDEX])]),
    ([(0, 1, 0), (0, 2, 0)], [(3, [_lib.OUT_S, _lib.OUT_O])]),
    ([(0, 0, 9), (9, 0, 0), (0, 9, 0)], [(7, [_lib.OUT_S, _lib.OUT_P, _lib.OUT_O])]),
]


@pytest.mark.parametrize("n", [1, 8191, 8192, 8193, 1_000_003, 3_000_000])
def test_scan_streams_match_oracle(gpu, n):
    rng = np.random.default_rng(n)
    rows = rng.integers(1, 12, size=(n, 3), dtype=np.uint32)
    base = 12345 if n % 2 else 0
    ds = DeviceStore.upload(TripleChunk(rows.reshape(-1), base))
    for keys, streams in CASES:
        want = expected(rows, base, keys, streams)
        got = run(ds, keys, streams)
        for s, (g, w) in enumerate(zip(got, want)):
            for a, b in zip(g, w):
                np.testing.assert_array_equal(a, b, err_msg=f"keys={keys} stream={s}")


def test_scan_selectivity_extremes(gpu):
    n = 2_000_000
    rows = np.ones((n, 3), dtype=np.uint32)
    rows[::3, 1] = 2
    ds = DeviceStore.upload(TripleChunk(rows.reshape(-1), 0))
    for key, cnt in (((0, 1, 0), n - len(rows[::3])), ((0, 2, 0), len(rows[::3])), ((0, 5, 0), 0),
                     ((1, 1, 1), n - len(rows[::3]))):
        (got,) = run(ds, [key], [(1, [_lib.OUT_INDEX])])
        assert len(got[0]) == cnt
        want = np.flatnonzero((rows[:, 1] == key[1]) & ((key[0] == 0) | (rows[:, 0] == key[0])))
        np.testing.assert_array_equal(got[0], want)


def test_capacity_hints_exact_small_and_large(gpu):
    """Hint mode (no mid-scan sync): exact, too small (re-emit) and too large
    hints all give the exact oracle result; dense and sparse tiles."""
    rng = np.random.default_rng(7)
    n = 1_500_000
    rows = rng.integers(1, 40, size=(n, 3), dtype=np.uint32)
    rows[: n // 3, 1] = 5  # dense region for p=5
    ds = DeviceStore.upload(TripleChunk(rows.reshape(-1), 0))
    hist = ds.predicate_counts()
    assert int(hist[5]) == int(np.sum(rows[:, 1] == 5))
    for p in (5, 7, 39):
        want = np.flatnonzero(rows[:, 1] == p)
        for hint in (int(hist[p]), max(1, int(hist[p]) // 3), int(hist[p]) * 2 + 5):
            spec = _lib.ScanSpec()
            spec.n_keys = 1
            spec.keys[0][:] = (0, p, 0)
            spec.n_streams = 1
            st = spec.streams[0]
            st.select = 1
            st.n_out = 3
            st.out[0], st.out[1], st.out[2] = _lib.OUT_S, _lib.OUT_O, _lib.OUT_INDEX
            st.capacity_hint = hint
            (t,) = _lib.run_scan(ds.handle, spec)
            assert t.n_rows == len(want)
            np.testing.assert_array_equal(t.column(2), want)
            np.testing.assert_array_equal(t.column(0), rows[want, 0])
            np.testing.assert_array_equal(t.column(1), rows[want, 2])
            t.free()
