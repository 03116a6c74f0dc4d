"""GPU: deferred row counts of TIDQ_SCAN_ASYNC scans.  Results queued back to
back resolve to the synchronous results; pending tables can be freed,
downloaded, joined and counted in any order; exhausting the pinned count
slots falls back to synchronous scans."""

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


@pytest.fixture(scope="module")
def store(gpu):
    n, n_p, n_e = 500_000, 50, 30_000
    ds = DeviceStore.generate(n, seed=13, n_p=n_p, n_e=n_e)
    chunk = TripleChunk(ds.download().reshape(-1), 0)
    return ds, chunk, SynthDictionary(n_p, n_e)


def test_async_results_match(gpu, store):
    ds, chunk, d = store
    qs = [plan.compile_query([plan.Group([plan.pattern("?s", P.format(r), "?o")], [])], d) for r in range(1, 30)]
    pending = [Q.evaluate_query_device(q, ds, d, row_cap=None) for q in qs]  # nothing resolved yet
    for q, t in reversed(list(zip(qs, pending))):  # resolve out of order
        want = oq.evaluate_query(q, chunk, d, row_cap=None)
        np.testing.assert_array_equal(table_rows(t.download()), want.rows())


def test_free_and_join_pending(gpu, store):
    ds, chunk, d = store
    q1 = plan.compile_query([plan.Group([plan.pattern("?s", P.format(2), "?o")], [])], d)
    for _ in range(50):  # freed while still in flight
        Q.evaluate_query_device(q1, ds, d).t.free()
    q2 = plan.compile_query([plan.Group([plan.pattern("?s", P.format(2), "?o"),
                                         plan.pattern("?o", P.format(3), "?z")], [])], d)
    got = Q.evaluate_query(q2, ds, d, row_cap=None)
    np.testing.assert_array_equal(table_rows(got), oq.evaluate_query(q2, chunk, d, row_cap=None).rows())


def test_slot_exhaustion_falls_back(gpu, store):
    ds, chunk, d = store
    q = plan.compile_query([plan.Group([plan.pattern("?s", P.format(7), "?o")], [])], d)
    want = oq.evaluate_query(q, chunk, d, row_cap=None).n_rows
    held = [Q.evaluate_query_device(q, ds, d, row_cap=None) for _ in range(4200)]  # > 4096 count slots
    assert all(t.n_rows == want for t in held)
    for t in held:
        t.t.free()


def test_mixed_queries_back_to_back(gpu, store):
    """Stars, chains, FILTERs, UNIONs and DISTINCTs queued back to back (async
    scans, chained operator launches), resolved only at the end, every result
    exact vs the oracle."""
    ds, chunk, d = store
    rng = np.random.default_rng(17)
    names = ["x", "y", "z", "w"]
    qs = []
    for i in range(60):
        kind = i % 4
        ranks = [int(r) for r in rng.choice(np.arange(1, 20), size=3, replace=False)]
        if kind == 0:  # star
            pats = [plan.pattern("?s", P.format(r), f"?o{j}") for j, r in enumerate(ranks[:2 + i % 2])]
            q = plan.compile_query([plan.Group(pats, [])], d)
        elif kind == 1:  # chain with FILTER
            pats = [plan.pattern(f"?{names[j]}", P.format(r), f"?{names[j + 1]}") for j, r in enumerate(ranks[:2])]
            q = plan.compile_query([plan.Group(pats, [plan.Filter("y", "7$")])], d)
        elif kind == 2:  # UNION bag / DISTINCT
            groups = [plan.Group([plan.pattern("?s", P.format(r), "?o")], []) for r in ranks]
            q = plan.compile_query(groups, d, distinct=bool(i % 3), projection=["s"] if i % 2 else None)
        else:  # star x3 (semi-join reduced) with projection
            pats = [plan.pattern("?s", P.format(r), f"?o{j}") for j, r in enumerate(ranks)]
            q = plan.compile_query([plan.Group(pats, [])], d, distinct=True, projection=["s", "o0"])
        qs.append(q)
    pending = [Q.evaluate_query_device(q, ds, d, row_cap=None) for q in qs]
    for q, t in zip(qs, pending):
        want = oq.evaluate_query(q, chunk, d, row_cap=None)
        got = t.download()
        assert got.columns == want.columns
        np.testing.assert_array_equal(table_rows(got), want.rows())
