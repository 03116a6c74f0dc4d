"""GPU: BASELINE configs[0] (C1) bit-exact against the reference.

The 1M-triple store (seed 1, n_p 10^4, n_e 10^5) is generated on the device;
its SHA-256 must equal the one recorded when the reference ran on the numpy
twin (tests/golden/make_golden.py), and every C1 query — ?s P_10 ?o (the
north star's bit-exact anchor) plus the C2-C5 shapes at C1 size — must return
the reference's rows in the reference's order, through the resident store,
the host-chunk operator path, and the .tid path."""

import hashlib

import numpy as np
import pytest

from helpers import plan_from_json, table_rows
from paper_1807_01409_b200 import query_ops as Q
from paper_1807_01409_b200.store import DeviceStore, TripleChunk, write_tid
from paper_1807_01409_b200.synth import SynthDictionary

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1(gpu, golden):
    meta, arrays = golden
    d = meta["dataset_C1"]
    ds = DeviceStore.generate(d["n"], seed=d["seed"], n_p=d["n_p"], n_e=d["n_e"])
    rows = ds.download()
    assert hashlib.sha256(rows.tobytes()).hexdigest() == d["rows_sha256"]
    yield ds, rows, SynthDictionary(d["n_p"], d["n_e"]), meta["c1"], arrays
    ds.free()


@pytest.mark.parametrize("mode", ["resident", "chunk", "tid"])
def test_c1_queries_bit_exact(c1, mode, tmp_path):
    ds, rows, dictionary, cases, arrays = c1
    if mode == "resident":
        store = ds
    elif mode == "chunk":
        store = TripleChunk(rows.reshape(-1), 0)
    else:
        store = str(tmp_path / "c1.tid")
        write_tid(rows, store)
    assert len(cases) >= 20
    for case in cases:
        t = Q.evaluate_query(plan_from_json(case["plan"]), store, dictionary, row_cap=case["row_cap"])
        assert t.columns == case["columns"], case["name"]
        want = arrays[case["result"]]
        assert t.n_rows == case["n_rows"], case["name"]
        np.testing.assert_array_equal(table_rows(t).reshape(want.shape), want, err_msg=case["name"])


def test_c1_queries_reduced_and_uncapped(c1):
    """row_cap=None takes the semi-join-reduced star path; same rows."""
    ds, _rows, dictionary, cases, arrays = c1
    for case in cases:
        t = Q.evaluate_query(plan_from_json(case["plan"]), ds, dictionary, row_cap=None)
        want = arrays[case["result"]]
        np.testing.assert_array_equal(table_rows(t).reshape(want.shape), want, err_msg=case["name"])
