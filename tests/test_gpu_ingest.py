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


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_load_shard_ranges_equal_read_chunks(gpu, tmp_path, world):
    """Row-range (shard) loads: rank g's store holds the file's rows
    [lo_g, hi_g) with global indices lo_g..; concatenated in rank order they
    equal read_chunks' rows and base indices, and per-shard scans
    concatenate to the whole-file scan (chunk invariance)."""
    from paper_1807_01409_b200.distributed import shard_bounds
    from paper_1807_01409_b200.store import read_chunks

    n = 1_000_003
    ds0 = DeviceStore.generate(n, seed=9, n_p=40, n_e=50_000)
    rows = ds0.download()
    ds0.free()
    p = tmp_path / "sh.tid"
    write_tid(rows, p)
    whole = [c for c in read_chunks(p, chunk_triples=n)][0]
    keys = [K.PatternKey(0, 3, 0), K.PatternKey(0, 7, 0)]
    want_i, want_m = osc.search_multi(whole, keys)
    parts, idx, marks = [], [], []
    for r in range(world):
        sh = DeviceStore.load_shard(p, r, world)
        lo, hi = shard_bounds(n, world, r)
        assert sh.base_index == lo and len(sh) == hi - lo
        parts.append(sh.download())
        res = K.search_multi(sh, keys)
        idx.append(res.indices)
        marks.append(res.values)
        sh.free()
    np.testing.assert_array_equal(np.concatenate(parts), rows)
    np.testing.assert_array_equal(np.concatenate(idx), want_i)
    np.testing.assert_array_equal(np.concatenate(marks), want_m)
    # an explicit range with a base offset, a range clamped at the end, an empty range
    st = DeviceStore.load(p, lo=10, n=5, base_index=100)
    assert st.base_index == 110 and len(st) == 5
    np.testing.assert_array_equal(st.download(), rows[10:15])
    st = DeviceStore.load(p, lo=n - 2, n=10)
    np.testing.assert_array_equal(st.download(), rows[n - 2:])
    assert len(DeviceStore.load(p, lo=n, n=10)) == 0
    with pytest.raises(ValueError):
        DeviceStore.load(p, lo=n + 1, n=1)
