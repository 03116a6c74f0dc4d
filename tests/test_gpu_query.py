"""GPU parity of the query operators through the C ABI against the reference's
golden outputs (bit-exact rows AND row order) and the oracle."""

import numpy as np
import pytest

from helpers import IdDictionary, plan_from_json, sorted_rows, table_rows
from oracle import query as oq
from oracle import scan as osc
from paper_1807_01409_b200 import query_ops as Q
from paper_1807_01409_b200.errors import DisconnectedPatterns, ResourceLimit
from paper_1807_01409_b200.store import DeviceStore, TripleChunk
from paper_1807_01409_b200.synth import SynthDictionary

pytestmark = pytest.mark.gpu


def dataset(meta, arrays, name):
    if name == "a":
        d = meta["dataset_a"]
        return TripleChunk(arrays[d["data"]].reshape(-1), 0), SynthDictionary(d["n_p"], d["n_e"])
    d = meta[f"dataset_{name}"]  # b, c, d: dense x.org ID spaces
    return TripleChunk(arrays[d["data"]].reshape(-1), 0), IdDictionary(d["max_id"])


@pytest.mark.parametrize("resident", [True, False])
def test_evaluate_query_golden(gpu, golden, resident):
    meta, arrays = golden
    stores = {}
    for case in meta["query"]:
        chunk, dictionary = dataset(meta, arrays, case["dataset"])
        if resident:
            store = stores.setdefault(case["dataset"], DeviceStore.upload(chunk))
        else:
            store = chunk
        plan = plan_from_json(case["plan"])
        if "error" in case:
            with pytest.raises(Exception) as ei:
                Q.evaluate_query(plan, store, dictionary, row_cap=case["row_cap"])
            assert type(ei.value).__name__ == case["error"], case["name"]
            continue
        qt = Q.QueryTimings()
        t = Q.evaluate_query(plan, store, dictionary, row_cap=case["row_cap"], timings=qt)
        assert t.columns == case["columns"], case["name"]
        want = arrays[case["result"]]
        got = table_rows(t)
        assert t.n_rows == case["n_rows"], case["name"]
        np.testing.assert_array_equal(got.reshape(want.shape), want, err_msg=case["name"])
        assert qt.search >= 0 and qt.join >= 0


def test_evaluate_query_chunked_store(gpu, golden, tmp_path):
    """chunk invariance: a .tid path read in 997-triple
    chunks gives the same rows in the same order."""
    from paper_1807_01409_b200.store import write_tid

    meta, arrays = golden
    chunk, dictionary = dataset(meta, arrays, "a")
    p = tmp_path / "a.tid"
    write_tid(chunk.rows, p)
    for case in meta["query"]:
        if case["dataset"] != "a" or "error" in case or case["name"] not in (
                "single_pp", "union4_distinct", "star3", "chain2_filter", "os_join", "union_unbound"):
            continue
        plan = plan_from_json(case["plan"])
        t = Q.evaluate_query(plan, str(p), dictionary, chunk_triples=997, row_cap=case["row_cap"])
        np.testing.assert_array_equal(table_rows(t).reshape(arrays[case["result"]].shape),
                                      arrays[case["result"]], err_msg=case["name"])


def test_merge_join_golden(gpu, golden):
    meta, arrays = golden
    for case in meta["merge_join"]:
        got = Q.merge_join(arrays[case["left"]], arrays[case["right"]])
        assert got.dtype == np.int64
        np.testing.assert_array_equal(got.reshape(-1, 2), arrays[case["pairs"]].reshape(-1, 2),
                                      err_msg=case["name"])


def test_merge_join_random_vs_nested_loop(gpu):
    rng = np.random.default_rng(3)
    for _ in range(20):
        lk = rng.integers(1, 30, size=int(rng.integers(0, 800))).astype(np.uint32)
        rk = rng.integers(1, 30, size=int(rng.integers(0, 800))).astype(np.uint32)
        got = Q.merge_join(lk, rk)
        want = np.argwhere(lk[:, None] == rk[None, :]) if len(lk) and len(rk) else np.empty((0, 2))
        np.testing.assert_array_equal(sorted_rows(got.reshape(-1, 2)), sorted_rows(want.reshape(-1, 2)))
        np.testing.assert_array_equal(got.reshape(-1, 2), oq.merge_join(lk, rk).reshape(-1, 2))


def test_project_distinct_and_union(gpu):
    rng = np.random.default_rng(4)
    for ncols in (1, 2, 3, 5):
        cols = [f"v{i}" for i in range(ncols)]
        data = {c: rng.integers(1, 4, size=3000).astype(np.uint32) for c in cols}
        t = Q.BindingTable(cols, data)
        for proj in (None, cols[:1], cols[::-1]):
            got = Q.project_distinct(t, proj, True)
            want = oq.project_distinct(oq.Table(cols, data), proj, True)
            assert got.columns == want.columns
            np.testing.assert_array_equal(table_rows(got), want.rows())
    same = Q.BindingTable(["a"], {"a": np.full(100, 7, np.uint32)})
    assert Q.project_distinct(same, None, True).n_rows == 1
    with pytest.raises(KeyError):
        Q.project_distinct(same, ["zz"], False)
    t1 = Q.BindingTable(["a", "b"], {"a": np.arange(1, 4, dtype=np.uint32), "b": np.arange(4, 7, dtype=np.uint32)})
    t2 = Q.BindingTable(["c", "a"], {"c": np.arange(9, 11, dtype=np.uint32), "a": np.arange(20, 22, dtype=np.uint32)})
    u = Q.evaluate_union([t1, t2])
    assert u.columns == ["a", "b", "c"] and u.n_rows == 5
    np.testing.assert_array_equal(u.data["b"], [4, 5, 6, 0, 0])
    np.testing.assert_array_equal(u.data["c"], [0, 0, 0, 9, 10])


def test_apply_filter_and_pattern_table(gpu, golden):
    meta, arrays = golden
    chunk, dictionary = dataset(meta, arrays, "a")
    rows = chunk.rows[chunk.rows[:, 1] == 1]
    from paper_1807_01409_b200 import plan

    pat = plan.pattern("?s", "<http://example.org/p/1>", "?o")
    bt = Q.pattern_table(pat, pat.var_slots(), rows)
    want = oq.pattern_table(pat, pat.var_slots(), rows)
    np.testing.assert_array_equal(table_rows(bt), want.rows())
    for rx in ("7$", "e/1", "^http", "zzz"):
        got = Q.apply_filter(bt, "o", rx, dictionary)
        exp = oq.apply_filter(want, "o", rx, dictionary)
        np.testing.assert_array_equal(table_rows(got), exp.rows())
    rep = plan.pattern("?x", "?p", "?x")
    allrows = chunk.rows
    got = Q.pattern_table(rep, rep.var_slots(), allrows)
    exp = oq.pattern_table(rep, rep.var_slots(), allrows)
    np.testing.assert_array_equal(table_rows(got), exp.rows())


def test_scan_patterns_vs_oracle(gpu, golden):
    meta, arrays = golden
    chunk, dictionary = dataset(meta, arrays, "a")
    for case in meta["query"][:12]:
        plan = plan_from_json(case["plan"])
        got = Q.scan_patterns(plan.groups, chunk)
        want = osc.scan_patterns(plan.groups, chunk)
        for g_got, g_want in zip(got, want):
            for a, b in zip(g_got, g_want):
                np.testing.assert_array_equal(a, b)


def test_join_group_and_errors(gpu, golden):
    meta, arrays = golden
    chunk, dictionary = dataset(meta, arrays, "a")
    qs = {q["name"]: q for q in meta["query"]}
    plan = plan_from_json(qs["star3"]["plan"])
    rows = osc.scan_patterns(plan.groups, chunk)[0]
    got = Q.join_group(plan.groups[0], rows, dictionary)
    np.testing.assert_array_equal(table_rows(got), arrays[qs["star3"]["result"]])
    with pytest.raises(ResourceLimit):
        Q.join_group(plan.groups[0], rows, dictionary, row_cap=10)
    with pytest.raises(DisconnectedPatterns):
        Q.evaluate_query(plan_from_json(qs["disconnected"]["plan"]), chunk, dictionary)
    with pytest.raises(ValueError):
        Q.evaluate_query(plan, chunk, dictionary, workers=0)
