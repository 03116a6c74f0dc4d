"""GPU: native .tid ingest (tidq_store_load_tid) — §8f row 1.  The loaded
store equals the reference's read_all; header/truncation errors are the
reference's (store.py:107-146); queries on a path equal the oracle."""

import struct

import numpy as np
import pytest

from oracle import query as oq
from oracle import scan as osc
from paper_1807_01409_b200 import kernel as K
from paper_1807_01409_b200 import plan
from paper_1807_01409_b200 import query_ops as Q
from paper_1807_01409_b200.errors import BadMagic, BadVersion, TruncatedFile
from paper_1807_01409_b200.store import DeviceStore, TripleChunk, read_all, write_tid
from paper_1807_01409_b200.synth import SynthDictionary

from helpers import table_rows

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [0, 1, 5, 4099, 9_000_001])
def test_load_equals_read_all(gpu, tmp_path, n):
    rng = np.random.default_rng(n)
    rows = rng.integers(1, 2**32 - 1, size=(n, 3), dtype=np.uint64).astype(np.uint32)
    p = tmp_path / "s.tid"
    write_tid(rows, p)
    ds = DeviceStore.load(p, base_index=7)
    assert len(ds) == n and ds.base_index == 7
    np.testing.assert_array_equal(ds.download(), read_all(p).rows)


def test_load_errors(gpu, tmp_path):
    p = tmp_path / "bad.tid"
    p.write_bytes(b"XXXX" + struct.pack("<IQ", 1, 0))
    with pytest.raises(BadMagic):
        DeviceStore.load(p)
    p.write_bytes(b"TID1" + struct.pack("<IQ", 2, 0))
    with pytest.raises(BadVersion):
        DeviceStore.load(p)
    p.write_bytes(b"TID1" + struct.pack("<IQ", 1, 5) + np.arange(1, 13, dtype="<u4").tobytes())
    with pytest.raises(TruncatedFile):
        DeviceStore.load(p)
    p.write_bytes(b"TID1"[:3])
    with pytest.raises(TruncatedFile):
        DeviceStore.load(p)
    with pytest.raises(FileNotFoundError):
        DeviceStore.load(tmp_path / "missing.tid")
    with pytest.raises(ValueError):
        K.search_file(p, K.PatternKey(0, 1, 0), chunk_triples=0)


def test_path_queries_native_and_chunked(gpu, tmp_path, monkeypatch):
    n, n_p, n_e = 300_000, 30, 20_000
    ds = DeviceStore.generate(n, seed=5, n_p=n_p, n_e=n_e)
    rows = ds.download()
    chunk = TripleChunk(rows.reshape(-1), 0)
    p = tmp_path / "g.tid"
    write_tid(rows, p)
    d = SynthDictionary(n_p, n_e)
    P = "<http://example.org/p/{}>"
    q = plan.compile_query([plan.Group([plan.pattern("?s", P.format(2), "?o"),
                                        plan.pattern("?o", P.format(3), "?z")],
                                       [plan.Filter("z", "1$")])], d)
    want = oq.evaluate_query(q, chunk, d, row_cap=None)
    keys = [K.PatternKey(0, 2, 0), K.PatternKey(0, 0, rows[10, 2])]
    wi, wm = osc.search_multi(chunk, keys)
    for fits in (True, False):  # whole-file native load, and the chunked fallback
        monkeypatch.setattr(DeviceStore, "fits", staticmethod(lambda path, device=None, f=fits: f))
        got = Q.evaluate_query(q, str(p), d, row_cap=None, chunk_triples=70_001)
        assert got.columns == want.columns
        np.testing.assert_array_equal(table_rows(got), want.rows())
        r = K.search_file(p, keys, chunk_triples=65_537)
        np.testing.assert_array_equal(r.indices, wi)
        np.testing.assert_array_equal(r.values, wm)
