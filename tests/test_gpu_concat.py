"""GPU: TIDQ_SCAN_CONCAT — a UNION of single-pattern branches scanned into
one table (stream order = branch order), against the oracle; the C-ABI
contract (empty tables for streams 1.., hint overflow re-emit, type checks)."""

import numpy as np
import pytest

from helpers import table_rows
from oracle import query as oq
from paper_1807_01409_b200 import _lib, plan
from paper_1807_01409_b200 import query_ops as Q
from paper_1807_01409_b200.store import DeviceStore, TripleChunk
from paper_1807_01409_b200.synth import SynthDictionary

pytestmark = pytest.mark.gpu
P = "<http://example.org/p/{}>"
E = "<http://example.org/e/{}>"


@pytest.fixture(scope="module")
def store(gpu):
    n, n_p, n_e = 1_500_000, 40, 20_000
    ds = DeviceStore.generate(n, seed=21, n_p=n_p, n_e=n_e)
    chunk = TripleChunk(ds.download().reshape(-1), 0)
    return ds, chunk, SynthDictionary(n_p, n_e)


def _check(q, ds, chunk, d):
    got = Q.evaluate_query(q, ds, d, row_cap=None)
    want = oq.evaluate_query(q, chunk, d, row_cap=None)
    assert got.columns == want.columns
    np.testing.assert_array_equal(table_rows(got), want.rows())


@pytest.mark.parametrize("proj,distinct", [(None, False), (["s"], False), (["s"], True), (["o", "s"], True)])
def test_concat_unions_vs_oracle(store, proj, distinct):
    ds, chunk, d = store
    # repeated branch (shared key), a dense and a sparse predicate, 3..12 branches
    for preds in ([3, 3], [1, 7, 2], [5, 9, 11, 13, 17, 19, 23, 29, 31, 37, 2, 4]):
        groups = [plan.Group([plan.pattern("?s", P.format(r), "?o")], []) for r in preds]
        q = plan.compile_query(groups, d, distinct=distinct, projection=proj)
        assert Q._concat_union(q, ds)
        _check(q, ds, chunk, d)


def test_concat_with_repeated_variable_and_bound_subject(store):
    """A branch ?s P ?s (equality predicate in the mark) and a branch with a
    bound object share the column list [s] after projection."""
    ds, chunk, d = store
    groups = [plan.Group([plan.pattern("?s", P.format(4), "?s")], []),
              plan.Group([plan.pattern("?s", P.format(6), "?o")], []),
              plan.Group([plan.pattern("?s", P.format(8), E.format(3))], [])]
    q = plan.compile_query(groups, d, projection=["s"])
    assert Q._concat_union(q, ds)
    _check(q, ds, chunk, d)


def test_not_concat_when_columns_differ(store):
    ds, chunk, d = store
    groups = [plan.Group([plan.pattern("?s", P.format(4), "?o")], []),
              plan.Group([plan.pattern("?x", P.format(6), "?o")], [])]
    q = plan.compile_query(groups, d)
    assert not Q._concat_union(q, ds)
    _check(q, ds, chunk, d)


def test_concat_pending_results_resolve_in_any_order(store):
    ds, chunk, d = store
    qs = [plan.compile_query([plan.Group([plan.pattern("?s", P.format(r + k), "?o")], []) for k in range(3)], d)
          for r in range(1, 20)]
    pending = [Q.evaluate_query_device(q, ds, d, row_cap=None) for q in qs]
    for q, t in reversed(list(zip(qs, pending))):
        np.testing.assert_array_equal(table_rows(t.download()),
                                      oq.evaluate_query(q, chunk, d, row_cap=None).rows())


def _spec(preds, hints, outs=None):
    spec = _lib.ScanSpec()
    spec.n_keys = len(preds)
    spec.n_streams = len(preds)
    for s, p in enumerate(preds):
        spec.keys[s][:] = (0, p, 0)
        st = spec.streams[s]
        st.select = 1 << s
        o = outs[s] if outs else (_lib.OUT_S, _lib.OUT_O)
        st.n_out = len(o)
        for k, kind in enumerate(o):
            st.out[k] = kind
        st.capacity_hint = hints[s]
    spec.flags = _lib.SCAN_CONCAT
    return spec


def test_concat_abi_sync_and_overflow(store):
    """Synchronous TIDQ_SCAN_CONCAT with exact hints and with hints too small
    (the emit is re-run into a larger table); streams 1.. come back empty."""
    ds, chunk, d = store
    rows = chunk.data.reshape(-1, 3)
    preds = [2, 5, 5, 9]
    want = np.concatenate([rows[rows[:, 1] == p][:, [0, 2]] for p in preds])
    exact = [int((rows[:, 1] == p).sum()) for p in preds]
    for hints in (exact, [1] * len(preds), [e // 2 + 1 for e in exact]):
        tables = _lib.run_scan(ds.handle, _spec(preds, hints))
        try:
            assert tables[0].n_rows == len(want)
            assert all(t.n_rows == 0 for t in tables[1:])
            np.testing.assert_array_equal(np.stack([tables[0].column(0), tables[0].column(1)], 1), want)
        finally:
            for t in tables:
                t.free()


def test_concat_abi_rejects_bad_specs(store):
    ds, _, _ = store
    with pytest.raises(ValueError):  # no capacity hints
        _lib.run_scan(ds.handle, _spec([2, 3], [0, 0]))
    with pytest.raises(ValueError):  # output types differ (index vs subject)
        _lib.run_scan(ds.handle, _spec([2, 3], [5, 5], outs=[(_lib.OUT_INDEX,), (_lib.OUT_S,)]))
    with pytest.raises(ValueError):  # output counts differ
        _lib.run_scan(ds.handle, _spec([2, 3], [5, 5], outs=[(_lib.OUT_S,), (_lib.OUT_S, _lib.OUT_O)]))
    # the context is still usable
    tables = _lib.run_scan(ds.handle, _spec([2, 3], [10**7, 10**7]))
    for t in tables:
        t.free()
