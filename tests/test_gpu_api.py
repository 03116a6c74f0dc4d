"""GPU: the rest of the reference's operator API against reference-generated
golden vectors — build_relation / BindingRelation.prepare_for_join /
merge_join on relations (query_ops.py:94-177), evaluate_group
(query_ops.py:345-356) — and the reference's error contract where the device
path has shortcuts: ResourceLimit on UNREDUCED pair counts of star groups
(query_ops.py:321-324), FILTER errors (query_ops.py:245-246), and FILTER
bitmaps that follow a growing dictionary."""

import numpy as np
import pytest

from helpers import IdDictionary, plan_from_json, table_rows
from oracle import query as oq
from paper_1807_01409_b200 import plan
from paper_1807_01409_b200 import query_ops as Q
from paper_1807_01409_b200.errors import ResourceLimit
from paper_1807_01409_b200.store import DeviceStore, TripleChunk, write_tid

pytestmark = pytest.mark.gpu


def _pattern(p):
    return plan.TriplePattern(*[plan.Var(x["var"]) if "var" in x else plan.Term(x["term"]) for x in p])


def test_relations_golden(gpu, golden):
    meta, arrays = golden
    for case in meta["relation"]:
        pat = _pattern(case["pattern"])
        rows = arrays[case["rows"]]
        if "error" in case:
            with pytest.raises(ValueError):
                Q.build_relation(rows, pat, case["join_slot"])
            continue
        rel = Q.build_relation(rows, pat, case["join_slot"])
        np.testing.assert_array_equal(rel.key, arrays[case["key"]], err_msg=case["name"])
        for k, name in case["values"].items():
            np.testing.assert_array_equal(rel.values[k], arrays[name], err_msg=case["name"])
        prep = rel.prepare_for_join()
        assert prep.sorted and prep.prepare_for_join() is prep and len(prep) == len(rel)
        np.testing.assert_array_equal(prep.key, arrays[case["sorted_key"]], err_msg=case["name"])
        for k, name in case["sorted_values"].items():
            np.testing.assert_array_equal(prep.values[k], arrays[name], err_msg=case["name"])
        if "self_pairs" in case:
            np.testing.assert_array_equal(Q.merge_join(rel, prep), arrays[case["self_pairs"]],
                                          err_msg=case["name"])


def test_prepare_for_join_large_stable(gpu):
    rng = np.random.default_rng(3)
    key = rng.integers(1, 5000, size=300_000, dtype=np.uint32)
    vals = {"O": rng.integers(1, 1 << 31, size=len(key), dtype=np.uint32)}
    prep = Q.BindingRelation(key, vals).prepare_for_join()
    order = np.argsort(key, kind="stable")
    np.testing.assert_array_equal(prep.key, key[order])
    np.testing.assert_array_equal(prep.values["O"], vals["O"][order])


@pytest.mark.parametrize("resident", [True, False])
def test_evaluate_group_golden(gpu, golden, resident):
    meta, arrays = golden
    d = meta["dataset_b"]
    chunk = TripleChunk(arrays[d["data"]].reshape(-1), 0)
    dictionary = IdDictionary(d["max_id"])
    store = DeviceStore.upload(chunk) if resident else chunk
    for case in meta["group"]:
        cg = plan_from_json(case["plan"]).groups[0]
        # both the compiled group and the uncompiled AST group (compiled here)
        for group in (cg, plan.Group(cg.patterns, cg.filters)):
            if "error" in case:
                with pytest.raises(Exception) as ei:
                    Q.evaluate_group(group, store, dictionary, row_cap=case["row_cap"])
                assert type(ei.value).__name__ == case["error"], case["name"]
                continue
            t = Q.evaluate_group(group, store, dictionary, row_cap=case["row_cap"])
            assert t.columns == case["columns"], case["name"]
            want = arrays[case["result"]]
            np.testing.assert_array_equal(table_rows(t).reshape(want.shape), want, err_msg=case["name"])


def _star_counterexample():
    """Subject 10 has 4,000 x:1 and 4,000 x:2 triples and no x:3 triple: the
    reference's first merge_join yields 16,000,000+ pairs (> the default cap
    10^7) although the 3-way star's result is small."""
    rows = [np.column_stack([np.full(4000, 10), np.full(4000, 1), np.arange(100, 4100)]),
            np.column_stack([np.full(4000, 10), np.full(4000, 2), np.arange(5000, 9000)])]
    s = np.repeat(np.arange(11, 2011), 6)
    p = np.tile(np.repeat([1, 2, 3], 2), 2000)
    o = 10_000 + (s * 7 + p * 3 + np.tile([0, 1], 6000)) % 5000
    rows.append(np.column_stack([s, p, o]))
    data = np.concatenate(rows).astype(np.uint32)
    data = data[np.random.default_rng(1).permutation(len(data))]
    return TripleChunk(np.ascontiguousarray(data).reshape(-1), 0), IdDictionary(20_000)


def test_row_cap_unreduced_star(gpu, tmp_path):
    chunk, dictionary = _star_counterexample()
    q = plan.compile_query([plan.Group([plan.pattern("?s", "<http://x.org/1>", "?a"),
                                        plan.pattern("?s", "<http://x.org/2>", "?b"),
                                        plan.pattern("?s", "<http://x.org/3>", "?c")], [])], dictionary)
    with pytest.raises(oq.ResourceLimit):
        oq.evaluate_query(q, chunk, dictionary)  # the oracle agrees with the reference's contract
    path = tmp_path / "c.tid"
    write_tid(chunk.rows, path)
    ds = DeviceStore.upload(chunk)
    for store in (ds, chunk, [chunk], str(path)):
        with pytest.raises(ResourceLimit):
            Q.evaluate_query(q, store, dictionary)
        with pytest.raises(ResourceLimit):
            Q.evaluate_group(q.groups[0], store, dictionary)
    want = oq.evaluate_query(q, chunk, dictionary, row_cap=None).rows()
    assert len(want) == 2000 * 8
    for store in (ds, chunk):
        np.testing.assert_array_equal(table_rows(Q.evaluate_query(q, store, dictionary, row_cap=None)), want)
        np.testing.assert_array_equal(table_rows(Q.evaluate_query(q, store, dictionary, row_cap=16_008_000)), want)
        with pytest.raises(ResourceLimit):  # the first join's pair count is 16,000,000 + 8,000
            Q.evaluate_query(q, store, dictionary, row_cap=16_007_999)


def test_filter_errors_like_reference(gpu):
    import re

    d = IdDictionary(50)
    rows = np.array([[1, 2, 3], [4, 2, 5]], dtype=np.uint32)
    ds = DeviceStore.upload(TripleChunk(rows.reshape(-1), 0))
    bad = plan.compile_query([plan.Group([plan.pattern("?s", "<http://x.org/9>", "?o")],
                                         [plan.Filter("o", "(unclosed")])], d)
    with pytest.raises(re.error):  # no rows, but the reference compiles the regex first
        Q.evaluate_query(bad, ds, d)
    t = Q.BindingTable(["a"], {"a": np.array([1, 2], np.uint32)})
    with pytest.raises(KeyError):
        Q.apply_filter(t, "zz", "1", d)
    with pytest.raises(re.error):
        Q.apply_filter(Q.BindingTable(["a"], {"a": np.empty(0, np.uint32)}), "a", "(", d)


class _GrowingDictionary(IdDictionary):
    def __len__(self):
        return self.max_id


def test_fused_filter_follows_dictionary_growth(gpu):
    """A complete FILTER bitmap built for a smaller dictionary must not drop
    rows whose IDs were added later (stale complete_upto)."""
    d = _GrowingDictionary(20)
    q_rows = np.array([[1, 2, 3], [4, 2, 15]], dtype=np.uint32)
    ds = DeviceStore.upload(TripleChunk(q_rows.reshape(-1), 0))
    q = plan.compile_query([plan.Group([plan.pattern("?s", "<http://x.org/2>", "?o")],
                                       [plan.Filter("o", "5$")])], d)
    assert table_rows(Q.evaluate_query(q, ds, d)).tolist() == [[4, 15]]
    d.max_id = 40  # new terms, then a store holding them
    rows2 = np.array([[1, 2, 3], [4, 2, 15], [6, 2, 35], [7, 2, 36]], dtype=np.uint32)
    ds2 = DeviceStore.upload(TripleChunk(rows2.reshape(-1), 0))
    assert table_rows(Q.evaluate_query(q, ds2, d)).tolist() == [[4, 15], [6, 35]]
    # IDs beyond the dictionary: decoded (and rejected) like the reference
    rows3 = np.array([[1, 2, 45]], dtype=np.uint32)
    ds3 = DeviceStore.upload(TripleChunk(rows3.reshape(-1), 0))
    with pytest.raises(KeyError):
        Q.evaluate_query(q, ds3, d)
    with pytest.raises(KeyError):
        oq.evaluate_query(q, TripleChunk(rows3.reshape(-1), 0), d)
