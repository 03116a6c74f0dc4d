"""GPU: BASELINE.json configurations at their full sizes, checked through
size-independent properties (the oracle cannot run at 10^8-10^9 triples):

* C2 (100 M): every single-pattern scan returns exactly the predicate's
  histogram count, in strictly ascending triple order, and the sampled
  triples really carry the predicate;
* C3 (500 M): UNION (bag) row count = sum of the branch counts; DISTINCT ?s
  = the number of distinct subjects of the union, first occurrences in order;
* C4 (500 M): |A join B| on a shared variable = sum over keys of
  count_A(key) * count_B(key) for star and chain joins, and every output row
  joins (the shared column agrees with both inputs);
* C5 (2 B): the 3-way star count = sum of count_A * count_B * count_C.
"""

import numpy as np
import pytest

from paper_1807_01409_b200 import kernel as K
from paper_1807_01409_b200 import plan
from paper_1807_01409_b200 import query_ops as Q
from paper_1807_01409_b200.store import DeviceStore
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary

pytestmark = pytest.mark.gpu
P = "<http://example.org/p/{}>"


def _store(cfg):
    c = CONFIGS[cfg]
    return DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"]), \
        SynthDictionary(c["n_p"], c["n_e"])


def _pairs(a: np.ndarray, b: np.ndarray) -> int:
    ka, ca = np.unique(a, return_counts=True)
    kb, cb = np.unique(b, return_counts=True)
    common, ia, ib = np.intersect1d(ka, kb, assume_unique=True, return_indices=True)
    return int((ca[ia].astype(np.int64) * cb[ib]).sum())


def test_c2_scan_counts_order_and_predicate(gpu):
    ds, d = _store("C2")
    hist = ds.predicate_counts()
    rng = np.random.default_rng(0)
    for r in (1, 10, 100, 1000, 10000):
        res = K.search_chunk(ds, K.PatternKey(0, r, 0))
        assert len(res) == int(hist[r])
        assert np.all(np.diff(res.indices) > 0)
        assert np.all(res.values == 2)
        sample = res.indices[rng.integers(0, len(res), size=min(len(res), 2000))]
        assert np.all(ds.gather(sample)[:, 1] == r)
    ds.free()


def test_c3_union_and_distinct_properties(gpu):
    ds, d = _store("C3")
    hist = ds.predicate_counts()
    ranks = [2, 3, 4, 5]
    groups = [plan.Group([plan.pattern("?s", P.format(r), "?o")], []) for r in ranks]
    bag = Q.evaluate_query(plan.compile_query(groups, d), ds, d, row_cap=None)
    assert bag.n_rows == int(sum(hist[r] for r in ranks))
    dist = Q.evaluate_query(plan.compile_query(groups, d, distinct=True, projection=["s"]), ds, d, row_cap=None)
    s = bag.data["s"]
    u, first = np.unique(s, return_index=True)
    assert dist.n_rows == len(u)
    np.testing.assert_array_equal(dist.data["s"], s[np.sort(first)])  # first occurrences, in order
    ds.free()


@pytest.mark.parametrize("shape", ["star", "chain"])
def test_c4_join_counts(gpu, shape):
    ds, d = _store("C4")
    if shape == "star":
        a, b = plan.pattern("?s", P.format(3), "?o1"), plan.pattern("?s", P.format(5), "?o2")
        key_a, key_b, var = "s", "s", "s"
    else:
        a, b = plan.pattern("?x", P.format(3), "?y"), plan.pattern("?y", P.format(5), "?z")
        key_a, key_b, var = "o", "s", "y"
    ta = Q.evaluate_query(plan.compile_query([plan.Group([plan.pattern("?s", P.format(3), "?o")], [])], d),
                          ds, d, row_cap=None)
    tb = Q.evaluate_query(plan.compile_query([plan.Group([plan.pattern("?s", P.format(5), "?o")], [])], d),
                          ds, d, row_cap=None)
    want = _pairs(ta.data[key_a], tb.data[key_b])
    got = Q.evaluate_query(plan.compile_query([plan.Group([a, b], [])], d), ds, d, row_cap=None)
    assert got.n_rows == want
    keys_a = set(np.unique(ta.data[key_a]).tolist())
    sample = got.data[var][:: max(1, got.n_rows // 5000)]
    assert all(int(k) in keys_a for k in sample)
    ds.free()


def test_c5_star3_count(gpu):
    ds, d = _store("C5")
    cols = []
    for r in (5, 7, 11):
        t = Q.evaluate_query(plan.compile_query([plan.Group([plan.pattern("?s", P.format(r), "?o")], [])], d),
                             ds, d, row_cap=None)
        cols.append(t.data["s"])
    ks = [np.unique(c, return_counts=True) for c in cols]
    common = np.intersect1d(np.intersect1d(ks[0][0], ks[1][0]), ks[2][0])
    want_total = np.ones(len(common), dtype=np.int64)
    for k, c in ks:
        want_total *= c[np.searchsorted(k, common)]
    want = int(want_total.sum())
    q = plan.compile_query([plan.Group([plan.pattern("?s", P.format(r), f"?o{i}")
                                        for i, r in enumerate((5, 7, 11))], [])], d)
    got = Q.evaluate_query_device(q, ds, d, row_cap=None)
    assert got.n_rows == want
    got.t.free()
    ds.free()
