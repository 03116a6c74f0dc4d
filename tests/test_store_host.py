"""CPU suite: host side of the store (the .tid format, chunking, memory math)
against SPEC.md:180-200 known answers."""

import numpy as np
import pytest

from paper_1807_01409_b200 import store as S
from paper_1807_01409_b200.errors import BadMagic, BadVersion, InvariantViolation, TruncatedFile


def test_write_tid_sizes(tmp_path):
    p = tmp_path / "a.tid"
    assert S.write_tid([], p) == 0 and p.stat().st_size == 16
    tri = [(1, 2, 3), (4, 5, 6), (7, 8, 9), (1, 1, 1), (2, 2, 2)]
    assert S.write_tid(tri, p) == 5 and p.stat().st_size == 76


def test_read_chunks_7_by_3(tmp_path):
    p = tmp_path / "b.tid"
    rows = np.arange(1, 22, dtype=np.uint32).reshape(7, 3)
    S.write_tid(rows, p)
    chunks = list(S.read_chunks(p, 3))
    assert [c.triple_count for c in chunks] == [3, 3, 1]
    assert [c.base_index for c in chunks] == [0, 3, 6]
    np.testing.assert_array_equal(np.concatenate([c.data for c in chunks]), rows.reshape(-1))
    assert len(list(S.read_chunks(p, 100))) == 1
    with pytest.raises(ValueError):
        list(S.read_chunks(p, 0))


def test_errors(tmp_path):
    p = tmp_path / "c.tid"
    S.write_tid(np.ones((10, 3), np.uint32), p)
    raw = p.read_bytes()
    p.write_bytes(raw[:-12])
    with pytest.raises(TruncatedFile):
        list(S.read_chunks(p, 4))
    p.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(BadMagic):
        S.read_header(p)
    p.write_bytes(raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    with pytest.raises(BadVersion):
        S.read_header(p)
    p.write_bytes(raw[:10])
    with pytest.raises(TruncatedFile):
        S.read_header(p)
    with pytest.raises(InvariantViolation):
        S.as_id_array([(1, 0, 2)])
    with pytest.raises(InvariantViolation):
        S.as_id_array([(1, 2**32, 2)])


def test_device_memory_bytes():
    assert [S.device_memory_bytes(n) for n in (0, 3, 15, 3_000_000)] == [12, 28, 92, 16_000_012]
    with pytest.raises(ValueError):
        S.device_memory_bytes(4)
    assert S.chunk_triples_for_budget(S.DEFAULT_MEMORY_BUDGET) == 15_728_640


def test_read_all_empty(tmp_path):
    p = tmp_path / "d.tid"
    S.write_tid([], p)
    assert S.read_all(p).triple_count == 0


def test_decode_table_tsv():
    """decode_table (query_ops.py:402-423): ?-prefixed header, verbatim terms,
    empty cells for UNBOUND, LF after every line."""
    import numpy as np

    from helpers import IdDictionary
    from paper_1807_01409_b200 import query_ops as Q

    d = IdDictionary(100)
    t = Q.BindingTable(["s", "o"], {"s": np.array([3, 0, 3], np.uint32), "o": np.array([7, 9, 0], np.uint32)})
    assert Q.decode_table(t, d) == ("?s\t?o\n<http://x.org/3>\t<http://x.org/7>\n"
                                    "\t<http://x.org/9>\n<http://x.org/3>\t\n")
    assert Q.decode_table(Q.BindingTable(["s"], {"s": np.empty(0, np.uint32)}), d) == "?s\n"
