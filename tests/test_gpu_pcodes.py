"""The 16-bit predicate-code column (tidq_store_pcodes) and the interleaved
(s, o) column (tidq_store_so): scans of predicate-only passes stream the codes
instead of the uint32 predicate column, with key values translated to codes,
and emits needing both ?s and ?o gather (s, o) pairs.  Results must equal the
oracle's and the TIDQ_P16=0 / TIDQ_SO=0 (uint32 columns) results: single keys, UNIONs (lookup and
compare-per-stream mark kernels), absent predicates, predicate ID 0 in raw
chunks, repeated-variable and FILTER epilogues, partial last tiles."""

import numpy as np
import pytest

from oracle import scan as osc
from paper_1807_01409_b200 import kernel as K
from paper_1807_01409_b200.store import DeviceStore, TripleChunk

pytestmark = pytest.mark.gpu


def _store(rows, base=0):
    ch = TripleChunk(rows.reshape(-1), base)
    ds = DeviceStore.upload(ch)
    ds.predicate_counts()  # builds the code column
    ds._build_so()  # (normally after DeviceStore.SO_AFTER_SCANS scans)
    return ch, ds


def _check(ch, ds, keys, monkeypatch):
    want_i, want_m = osc.search_multi(ch, keys)
    for env in ("1", "0"):
        monkeypatch.setenv("TIDQ_P16", env)
        monkeypatch.setenv("TIDQ_SO", env)
        got = K.search_multi(ds, keys)
        np.testing.assert_array_equal(got.indices, want_i)
        np.testing.assert_array_equal(got.values, want_m)
        wi, wb = osc.search_chunk(ch, keys[0])
        g1 = K.search_chunk(ds, keys[0])
        np.testing.assert_array_equal(g1.indices, wi)
        np.testing.assert_array_equal(g1.values, wb)


@pytest.mark.parametrize("n", [1, 4095, 4097, 200_003])
def test_pcodes_predicate_keys(gpu, n, monkeypatch):
    rng = np.random.default_rng(n)
    rows = np.empty((n, 3), dtype=np.uint32)
    rows[:, 0] = rng.integers(1, 1000, n)
    rows[:, 1] = rng.choice(np.array([0, 7, 9, 300, 70_000, 5_000_000], dtype=np.uint32), n)  # sparse ID space
    rows[:, 2] = rng.integers(1, 1000, n)
    ch, ds = _store(rows, base=int(rng.integers(0, 2**33)))
    assert ds.pcodes and ds.so
    present = [int(v) for v in np.unique(rows[:, 1])]
    for keys in ([(0, present[-1], 0)],
                 [(0, 8, 0)],  # absent predicate
                 [(0, p, 0) for p in present],  # UNION of every predicate (lookup or compare kernels)
                 [(0, 9, 0), (0, 300, 0), (0, 8, 0), (0, 12345, 0)],  # present and absent mixed
                 [(0, 7, 0), (0, 9, 0)],
                 [(0, 0, 0), (0, 7, 0)]):  # all-triples key next to a predicate key
        _check(ch, ds, [K.PatternKey(*k) for k in keys], monkeypatch)
    ds.free()


def test_pcodes_with_epilogues(gpu, golden, monkeypatch):
    """golden evaluate_query cases (FILTER, repeated variables, UNION) with the
    code column built, vs the reference's rows, both column choices."""
    from helpers import IdDictionary, plan_from_json, table_rows
    from paper_1807_01409_b200 import query_ops as Q
    from paper_1807_01409_b200.synth import SynthDictionary

    meta, arrays = golden
    stores = {}
    for env in ("1", "0"):
        monkeypatch.setenv("TIDQ_P16", env)
        monkeypatch.setenv("TIDQ_SO", env)
        for case in meta["query"]:
            if "error" in case:
                continue
            name = case["dataset"]
            dd = meta["dataset_a" if name == "a" else f"dataset_{name}"]
            d = SynthDictionary(dd["n_p"], dd["n_e"]) if name == "a" else IdDictionary(dd["max_id"])
            if name not in stores:
                stores[name] = _store(arrays[dd["data"]])[1]
            t = Q.evaluate_query(plan_from_json(case["plan"]), stores[name], d, row_cap=case["row_cap"])
            want = arrays[case["result"]]
            assert t.columns == case["columns"], case["name"]
            np.testing.assert_array_equal(table_rows(t).reshape(want.shape), want, err_msg=case["name"])


def test_pcodes_errors(gpu):
    from paper_1807_01409_b200 import _lib

    rows = np.array([[1, 2, 3], [4, 5, 6]], dtype=np.uint32)
    ds = DeviceStore.upload(TripleChunk(rows.reshape(-1), 0))
    bad = np.array([5, 2], dtype=np.uint32)
    with pytest.raises(Exception):
        _lib.call("tidq_store_pcodes", ds.handle, _lib.ptr(bad), 2)
    ok = np.array([2, 5], dtype=np.uint32)
    _lib.call("tidq_store_pcodes", ds.handle, _lib.ptr(ok), 2)
    _lib.call("tidq_store_pcodes", ds.handle, 0, 0)  # drop
    got = K.search_multi(ds, [K.PatternKey(0, 5, 0)])
    assert list(got.indices) == [1]
    ds.free()


def test_so_built_after_repeated_scans(gpu):
    """The (s, o) pair column is built once a store has served
    DeviceStore.SO_AFTER_SCANS predicate scans; queries give the same rows
    before and after."""
    rng = np.random.default_rng(3)
    rows = rng.integers(1, 50, size=(30_000, 3), dtype=np.uint32)
    ch = TripleChunk(rows.reshape(-1), 0)
    ds = DeviceStore.upload(ch)
    keys = [K.PatternKey(0, 7, 0)]
    want_i, want_m = osc.search_multi(ch, keys)
    for i in range(DeviceStore.SO_AFTER_SCANS + 1):
        ds.predicate_counts()
        assert ds.so == (i + 1 >= DeviceStore.SO_AFTER_SCANS)
        got = K.search_multi(ds, keys)
        np.testing.assert_array_equal(got.indices, want_i)
        np.testing.assert_array_equal(got.values, want_m)
    ds.free()


@pytest.mark.parametrize("n_keys", [1, 2, 3, 5, 8])
def test_pcodes_fp16_compares_at_the_code_range_ends(gpu, n_keys, monkeypatch):
    """The multi-stream code mark compares codes as fp16 bit patterns (rank +
    0x400): a store with 29,990 distinct predicates puts the highest codes
    near the top of the normal fp16 range; UNIONs of the lowest, the highest
    and absent predicates must match the oracle with either compare."""
    rng = np.random.default_rng(n_keys)
    n = 400_000
    preds = np.arange(1, 29_991, dtype=np.uint32) * 3  # 29,990 distinct IDs
    rows = np.empty((n, 3), dtype=np.uint32)
    rows[:, 0] = rng.integers(1, 1000, n)
    rows[:, 1] = preds[rng.integers(0, len(preds), n)]
    rows[: len(preds), 1] = preds  # every predicate present
    rows[:, 2] = rng.integers(1, 1000, n)
    ch, ds = _store(rows)
    assert ds.pcodes
    picks = [int(preds[0]), int(preds[-1]), int(preds[-2]), 4, int(preds[1]), int(preds[-3]), 5, int(preds[7])]
    keys = [K.PatternKey(0, p, 0) for p in picks[:n_keys]]
    for f16 in ("1", "0"):
        monkeypatch.setenv("TIDQ_MARK_F16", f16)
        _check(ch, ds, keys, monkeypatch)
    ds.free()
