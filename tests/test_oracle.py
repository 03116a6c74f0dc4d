"""CPU suite: pin the oracle to the reference's own outputs (golden vectors made
by tests/golden/make_golden.py running /root/reference) and to SPEC.md's
known-answer examples.  No GPU needed."""

import numpy as np
import pytest

from helpers import IdDictionary, plan_from_json, sorted_rows, table_rows
from oracle import query as oq
from oracle import scan as osc
from paper_1807_01409_b200.kernel import PatternKey, accepts, match_bits
from paper_1807_01409_b200.store import TripleChunk
from paper_1807_01409_b200.synth import SynthDictionary


def chunk_of(arrays, case):
    return TripleChunk(arrays[case["data"]].reshape(-1), case["base"])


def test_truth_table(golden):
    meta, _ = golden
    assert len(meta["truth_table"]) == 64
    for mask, combo, bits, acc in meta["truth_table"]:
        key = PatternKey(*(10 + i if mask & (4 >> i) else 0 for i in range(3)))
        triple = tuple((10 + i) if combo & (4 >> i) else (20 + i) for i in range(3))
        assert match_bits(triple, key) == bits
        assert int(accepts(bits, key)) == acc


def test_spec_match_bits_examples():
    # SPEC.md:246-258
    assert match_bits((1, 2, 1), PatternKey(1, 2, 0)) == 6
    assert match_bits((5, 6, 7), PatternKey(5, 6, 7)) == 7
    assert match_bits((9, 9, 9), PatternKey()) == 0
    assert match_bits((31, 84, 77), PatternKey(0, 84, 0)) == 2
    assert accepts(6, PatternKey(1, 2, 0)) and not accepts(2, PatternKey(1, 2, 0))
    assert accepts(0, PatternKey())


def test_oracle_rule11():
    # SPEC.md:265-276
    rows = np.array([[76, 84, 56], [31, 84, 77], [56, 84, 78], [56, 84, 77], [44, 83, 2]], np.uint32)
    ch = TripleChunk(rows.reshape(-1), 0)
    idx, bits = osc.search_chunk(ch, PatternKey(0, 84, 0))
    assert idx.tolist() == [0, 1, 2, 3] and bits.tolist() == [2, 2, 2, 2]
    idx, bits = osc.search_chunk(ch, PatternKey(44, 83, 2))
    assert idx.tolist() == [4] and bits.tolist() == [7]
    idx, marks = osc.search_multi(TripleChunk(np.array([5, 6, 9], np.uint32), 0),
                                  [PatternKey(5, 0, 0), PatternKey(0, 6, 0)])
    assert idx.tolist() == [0] and marks.tolist() == [3]


@pytest.mark.parametrize("workers", [1, 3])
def test_oracle_search_multi_golden(golden, workers):
    meta, arrays = golden
    for case in meta["scan"]:
        keys = [PatternKey(*k) for k in case["keys"]]
        idx, marks = osc.search_multi(chunk_of(arrays, case), keys, workers)
        np.testing.assert_array_equal(idx, arrays[case["indices"]], err_msg=case["name"])
        np.testing.assert_array_equal(marks, arrays[case["marks"]], err_msg=case["name"])
        assert idx.dtype == np.int64 and marks.dtype == np.uint32


def test_oracle_search_chunk_golden(golden):
    meta, arrays = golden
    for case in meta["chunk"]:
        idx, bits = osc.search_chunk(chunk_of(arrays, case), PatternKey(*case["key"]))
        np.testing.assert_array_equal(idx, arrays[case["indices"]], err_msg=case["name"])
        np.testing.assert_array_equal(bits, arrays[case["bits"]], err_msg=case["name"])
        assert bits.dtype == np.uint8


def test_oracle_merge_join_golden(golden):
    meta, arrays = golden
    for case in meta["merge_join"]:
        pairs = oq.merge_join(arrays[case["left"]], arrays[case["right"]])
        np.testing.assert_array_equal(pairs.reshape(-1, 2), arrays[case["pairs"]].reshape(-1, 2),
                                      err_msg=case["name"])


def test_oracle_relationships_golden(golden):
    meta, _ = golden
    qs = {q["name"]: q for q in meta["query"]}
    for r in meta["relationships"]:
        plan = plan_from_json(qs[r["query"]]["plan"])
        got = oq.analyze_relationships(plan.groups[r["group"]].patterns)
        assert [list(x) for x in got] == r["rels"]


def _dataset(meta, arrays, name):
    if name == "a":
        d = meta["dataset_a"]
        return TripleChunk(arrays[d["data"]].reshape(-1), 0), SynthDictionary(d["n_p"], d["n_e"])
    d = meta[f"dataset_{name}"]  # b, c, d: dense x.org ID spaces
    return TripleChunk(arrays[d["data"]].reshape(-1), 0), IdDictionary(d["max_id"])


def test_oracle_evaluate_query_golden(golden):
    """Bit-exact (including row order) against the reference's evaluate_query."""
    meta, arrays = golden
    for case in meta["query"]:
        chunk, dictionary = _dataset(meta, arrays, case["dataset"])
        plan = plan_from_json(case["plan"])
        if "error" in case:
            with pytest.raises(Exception) as ei:
                oq.evaluate_query(plan, chunk, dictionary, row_cap=case["row_cap"])
            assert type(ei.value).__name__ == case["error"], case["name"]
            continue
        t = oq.evaluate_query(plan, chunk, dictionary, row_cap=case["row_cap"])
        assert t.columns == case["columns"], case["name"]
        want = arrays[case["result"]]
        got = table_rows(t)
        assert got.shape[0] == case["n_rows"], case["name"]
        np.testing.assert_array_equal(got.reshape(want.shape), want, err_msg=case["name"])
        np.testing.assert_array_equal(sorted_rows(got.reshape(want.shape)), sorted_rows(want))


def test_oracle_synth_matches_golden_dataset(golden):
    from oracle import synth as osynth
    from paper_1807_01409_b200.synth import zipf_cdf_table

    meta, arrays = golden
    d = meta["dataset_a"]
    data = osynth.generate(d["n"], seed=d["seed"], n_p=d["n_p"], n_e=d["n_e"],
                           cdf=zipf_cdf_table(d["n_p"]))
    np.testing.assert_array_equal(data, arrays[d["data"]])
    # Zipf: rank-1 predicate frequency ~ 1/H(50)
    frac = np.mean(data[:, 1] == 1)
    assert 0.20 < frac < 0.26
    assert data.min() >= 1 and data[:, 1].max() <= d["n_p"]
    assert data[:, [0, 2]].min() > d["n_p"] and data[:, [0, 2]].max() <= d["n_p"] + d["n_e"]


def _pattern_from_json(p):
    from paper_1807_01409_b200 import plan

    return plan.TriplePattern(*[plan.Var(x["var"]) if "var" in x else plan.Term(x["term"]) for x in p])


def test_oracle_relations_golden(golden):
    """build_relation / prepare_for_join / merge_join of relations (query_ops.py:94-177)."""
    meta, arrays = golden
    for case in meta["relation"]:
        pat = _pattern_from_json(case["pattern"])
        rows = arrays[case["rows"]]
        if "error" in case:
            with pytest.raises(ValueError):
                oq.build_relation(rows, pat, case["join_slot"])
            continue
        key, values = oq.build_relation(rows, pat, case["join_slot"])
        np.testing.assert_array_equal(key, arrays[case["key"]])
        assert sorted(values) == sorted(case["values"])
        skey, svals = oq.prepare_for_join(key, values)
        np.testing.assert_array_equal(skey, arrays[case["sorted_key"]])
        for k, name in case["sorted_values"].items():
            np.testing.assert_array_equal(svals[k], arrays[name])
        if "self_pairs" in case:
            np.testing.assert_array_equal(oq.merge_join(key, skey), arrays[case["self_pairs"]])


def test_oracle_evaluate_group_golden(golden):
    meta, arrays = golden
    chunk, dictionary = _dataset(meta, arrays, "b")
    for case in meta["group"]:
        cg = plan_from_json(case["plan"]).groups[0]
        if "error" in case:
            with pytest.raises(Exception) as ei:
                oq.evaluate_group(cg, chunk, dictionary, row_cap=case["row_cap"])
            assert type(ei.value).__name__ == case["error"]
            continue
        t = oq.evaluate_group(cg, chunk, dictionary, row_cap=case["row_cap"])
        assert t.columns == case["columns"]
        np.testing.assert_array_equal(t.rows().reshape(arrays[case["result"]].shape), arrays[case["result"]])


def test_oracle_c1_config_golden(golden):
    """BASELINE configs[0] (C1, 1M triples, seed 1): the oracle on the
    regenerated store reproduces the reference's own evaluate_query output
    (rows and order) for ?s P_10 ?o and the C2-C5 query shapes at C1 size."""
    import hashlib

    from oracle import synth as osynth
    from paper_1807_01409_b200.synth import zipf_cdf_table

    meta, arrays = golden
    d = meta["dataset_C1"]
    rows = osynth.generate(d["n"], seed=d["seed"], n_p=d["n_p"], n_e=d["n_e"], cdf=zipf_cdf_table(d["n_p"]))
    assert hashlib.sha256(rows.tobytes()).hexdigest() == d["rows_sha256"]
    chunk, dictionary = TripleChunk(rows.reshape(-1), 0), SynthDictionary(d["n_p"], d["n_e"])
    assert len(meta["c1"]) >= 20
    for case in meta["c1"]:
        t = oq.evaluate_query(plan_from_json(case["plan"]), chunk, dictionary, row_cap=case["row_cap"])
        assert t.columns == case["columns"], case["name"]
        want = arrays[case["result"]]
        np.testing.assert_array_equal(table_rows(t).reshape(want.shape), want, err_msg=case["name"])
