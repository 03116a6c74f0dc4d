"""GPU: table operators at multi-tile sizes and every radix digit width
(8/9/10-bit digits, 1..3 passes, u32 and packed u64 keys), against the oracle
— exact rows and order."""

import numpy as np
import pytest

from helpers import table_rows
from oracle import query as oq
from paper_1807_01409_b200 import plan
from paper_1807_01409_b200 import query_ops as Q
from paper_1807_01409_b200.store import DeviceStore, TripleChunk
from paper_1807_01409_b200.synth import SynthDictionary

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ncols,hi,n", [(1, 200, 300_000), (1, 2**20, 500_000), (1, 2**32 - 1, 200_000),
                                        (2, 50, 400_000), (2, 3000, 300_000), (2, 2**31, 100_000),
                                        (3, 40, 200_000), (4, 12, 100_000)])
def test_distinct_large(gpu, ncols, hi, n):
    rng = np.random.default_rng(ncols * 1000 + n)
    cols = [f"c{i}" for i in range(ncols)]
    data = {c: rng.integers(1, hi, size=n, dtype=np.uint64).astype(np.uint32) for c in cols}
    t = Q.BindingTable(cols, data)
    got = Q.project_distinct(t, cols, True)
    want = oq.project_distinct(oq.Table(cols, data), cols, True)
    np.testing.assert_array_equal(table_rows(got), want.rows())


@pytest.mark.parametrize("n", [400_001, 1_000_003])
def test_distinct_table_hot_keys_any_order(gpu, n):
    """The first-occurrence table (one narrow column): hot keys repeated
    across the whole table and inside warps, first occurrences late in the
    table, a row count off the keep bitmap's byte/word edges."""
    rng = np.random.default_rng(n)
    a = rng.integers(1, 1 << 20, size=n).astype(np.uint32)
    a[rng.integers(0, n, size=n // 4)] = 7           # one key ~25 % of the rows
    a[n - 40:] = np.arange(1 << 20, (1 << 20) + 40)   # keys first seen in the last rows
    a[rng.integers(0, n, size=1000)] = a[n - 3]       # ... and repeated before them
    a[:64] = 11                                       # a whole warp of one key
    for data in ({"a": a}, {"a": a[::-1].copy()}):
        got = Q.project_distinct(Q.BindingTable(["a"], data), ["a"], True)
        want = oq.project_distinct(oq.Table(["a"], data), ["a"], True)
        np.testing.assert_array_equal(table_rows(got), want.rows())


@pytest.mark.parametrize("n,hi", [(100_000, 100), (200_000, 50_000), (300_000, 2**30)])
def test_merge_join_large(gpu, n, hi):
    rng = np.random.default_rng(n + hi)
    lk = rng.integers(1, hi, size=n).astype(np.uint32)
    rk = rng.integers(1, hi, size=n // 3).astype(np.uint32)
    if hi <= 100:  # keep the cross product small
        lk = lk[:3000]
        rk = rk[:1000]
    got = Q.merge_join(lk, rk)
    want = oq.merge_join(lk, rk)
    np.testing.assert_array_equal(got.reshape(-1, 2), want.reshape(-1, 2))


def test_unique_and_filter_large(gpu):
    rng = np.random.default_rng(3)
    col = rng.integers(1, 200_000, size=700_000).astype(np.uint32)
    t = Q.DevTable.upload(["x"], {"x": col})
    np.testing.assert_array_equal(Q._dev_unique(t, "x"), np.unique(col))


def test_union_scan_projection_and_distinct_vs_oracle(gpu):
    """UNION of up to 8 ?P? branches (the multi-key one-column mark path),
    projections that drop dead columns, DISTINCT over 1 and 2 columns."""
    n, n_p, n_e = 2_000_000, 50, 40_000
    ds = DeviceStore.generate(n, seed=9, n_p=n_p, n_e=n_e)
    rows = ds.download()
    chunk = TripleChunk(rows.reshape(-1), 0)
    d = SynthDictionary(n_p, n_e)
    P = "<http://example.org/p/{}>"
    for k in (2, 4, 8):
        groups = [plan.Group([plan.pattern("?s", P.format(r), "?o")], []) for r in range(1, k + 1)]
        for proj, distinct in ((["s"], True), (["s", "o"], True), (["o"], False), (None, False)):
            q = plan.compile_query(groups, d, distinct=distinct, projection=proj)
            got = Q.evaluate_query(q, ds, d, row_cap=None)
            want = oq.evaluate_query(q, chunk, d, row_cap=None)
            assert got.columns == want.columns
            np.testing.assert_array_equal(table_rows(got), want.rows(), err_msg=f"{k} {proj} {distinct}")
    # mixed keys: ?P? and S?? in one union (general multi-key mark path)
    groups = [plan.Group([plan.pattern("?s", P.format(2), "?o")], []),
              plan.Group([plan.pattern(f"<http://example.org/e/{7}>", "?p", "?o")], [])]
    q = plan.compile_query(groups, d, distinct=True, projection=["o"])
    np.testing.assert_array_equal(table_rows(Q.evaluate_query(q, ds, d)),
                                  oq.evaluate_query(q, chunk, d).rows())


@pytest.mark.parametrize("shape", ["star", "chain"])
def test_joins_at_scale_vs_oracle(gpu, shape):
    """2- and 3-way star/chain joins with FILTER on a 2M-triple store: the
    sides are large enough for the semi-join reduction and the staged
    equal_range/expand paths; exact rows and order vs the oracle."""
    n, n_p, n_e = 2_000_000, 40, 200_000
    ds = DeviceStore.generate(n, seed=21, n_p=n_p, n_e=n_e)
    chunk = TripleChunk(ds.download().reshape(-1), 0)
    d = SynthDictionary(n_p, n_e)
    P = "<http://example.org/p/{}>"
    names = ["x", "y", "z", "w"]
    for k in (2, 3):
        ranks = [3, 5, 7][:k]
        if shape == "star":
            pats = [plan.pattern("?s", P.format(r), f"?o{i}") for i, r in enumerate(ranks)]
            flt = [plan.Filter("o0", "7$")]
        else:
            pats = [plan.pattern(f"?{names[i]}", P.format(r), f"?{names[i + 1]}") for i, r in enumerate(ranks)]
            flt = [plan.Filter("y", "3$")]
        for filters in ([], flt):
            q = plan.compile_query([plan.Group(pats, filters)], d)
            got = Q.evaluate_query(q, ds, d, row_cap=None)
            want = oq.evaluate_query(q, chunk, d, row_cap=None)
            assert got.columns == want.columns
            assert got.n_rows > 0
            np.testing.assert_array_equal(table_rows(got), want.rows(), err_msg=f"{shape} {k} {filters}")


def test_merge_join_skips_semi_filter_for_huge_ids(gpu):
    """keys above 2^31 disable the key-bitmap reduction; results unchanged"""
    rng = np.random.default_rng(5)
    lk = rng.integers(2**31, 2**32 - 1, size=80_000, dtype=np.uint64).astype(np.uint32)
    rk = np.concatenate([lk[::7], rng.integers(1, 2**32 - 1, size=20_000, dtype=np.uint64).astype(np.uint32)])
    np.testing.assert_array_equal(Q.merge_join(lk, rk).reshape(-1, 2), oq.merge_join(lk, rk).reshape(-1, 2))


@pytest.mark.parametrize("n", [600_000, 600_005, 65_541])
def test_distinct_two_columns_partition_and_skew(gpu, n):
    """DISTINCT over two columns: the hash-partition path (wide keys, many
    duplicates across the whole table; row counts off the keep bitmap's byte
    and word edges) and its fallback to the sort when one key repeats more
    often than a partition table holds."""
    rng = np.random.default_rng(77 + n)
    a = rng.integers(1, 2**31, size=n // 3, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(1, 2**31, size=n // 3, dtype=np.uint64).astype(np.uint32)
    idx = rng.integers(0, n // 3, size=n)  # every pair ~3 times, scattered
    for data in ({"x": a[idx], "y": b[idx]},
                 {"x": np.where(np.arange(n) % 3 == 0, np.uint32(5), a[idx]),
                  "y": np.where(np.arange(n) % 3 == 0, np.uint32(9), b[idx])}):  # (5, 9) x 200k
        t = Q.BindingTable(["x", "y"], data)
        got = Q.project_distinct(t, ["x", "y"], True)
        want = oq.project_distinct(oq.Table(["x", "y"], data), ["x", "y"], True)
        np.testing.assert_array_equal(table_rows(got), want.rows())


def test_semijoin_reduced_star_groups_vs_oracle(gpu):
    """Star groups (a variable in 3+ patterns) take the semi-join-reduced scan
    (local indices + join variables, tidq_tables_semijoin, late gather):
    SELECT *, a projection that drops non-join columns, DISTINCT, a UNION of
    two star groups, a repeated variable, and a star whose reduction leaves
    nothing — exact rows and order vs the oracle."""
    n, n_p, n_e = 1_500_000, 30, 60_000
    ds = DeviceStore.generate(n, seed=31, n_p=n_p, n_e=n_e)
    chunk = TripleChunk(ds.download().reshape(-1), 0)
    d = SynthDictionary(n_p, n_e)
    P = "<http://example.org/p/{}>"
    star = lambda ranks, sv="s": [plan.pattern(f"?{sv}", P.format(r), f"?o{i}") for i, r in enumerate(ranks)]
    cases = [
        ([plan.Group(star([2, 3, 5]), [])], False, None),
        ([plan.Group(star([2, 3, 5, 7]), [])], True, ["s", "o1"]),
        ([plan.Group(star([2, 4, 6]), []), plan.Group(star([3, 5, 8]), [])], False, ["s"]),
        ([plan.Group(star([2, 3]) + [plan.pattern("?s", P.format(9), "?s")], [])], False, None),
        ([plan.Group(star([28, 29, 30]), [])], False, None),
    ]
    for groups, distinct, proj in cases:
        q = plan.compile_query(groups, d, distinct=distinct, projection=proj)
        got = Q.evaluate_query(q, ds, d, row_cap=None)
        want = oq.evaluate_query(q, chunk, d, row_cap=None)
        assert got.columns == want.columns
        np.testing.assert_array_equal(table_rows(got), want.rows(), err_msg=str((distinct, proj)))


def test_queries_on_huge_term_ids(gpu):
    """IDs near 2^32 (the dictionary's MAX_ID range): joins, star groups and
    DISTINCT fall back from the ID-sized bitmaps and stay exact."""
    rng = np.random.default_rng(99)
    n = 200_000
    ents = rng.integers(2**32 - 5_000_000, 2**32 - 1, size=20_000, dtype=np.uint64).astype(np.uint32)
    preds = np.array([2**32 - 7, 2**32 - 8, 2**32 - 9, 11], dtype=np.uint32)
    rows = np.stack([rng.choice(ents, n), rng.choice(preds, n), rng.choice(ents, n)], axis=1).astype(np.uint32)
    chunk = TripleChunk(rows.reshape(-1).copy(), 0)
    ds = DeviceStore.upload(chunk)

    class D:
        def lookup(self, lex):
            return int(lex[len("<http://x.org/"):-1])

        def decode_lexical(self, i):
            return f"<http://x.org/{i}>"

    d = D()
    P = "<http://x.org/{}>"
    p0, p1, p2 = (int(x) for x in preds[:3])
    star = [plan.pattern("?s", P.format(p), f"?o{i}") for i, p in enumerate((p0, p1, p2))]
    chain = [plan.pattern("?x", P.format(p0), "?y"), plan.pattern("?y", P.format(p1), "?z")]
    for groups, distinct, proj in (([plan.Group(star, [])], False, None),
                                   ([plan.Group(chain, [])], True, ["y"])):
        q = plan.compile_query(groups, d, distinct=distinct, projection=proj)
        got = Q.evaluate_query(q, ds, d, row_cap=None)
        want = oq.evaluate_query(q, chunk, d, row_cap=None)
        assert got.columns == want.columns
        np.testing.assert_array_equal(table_rows(got), want.rows())


@pytest.mark.parametrize("n", [3000, 60_000])
def test_join_of_join_outputs(gpu, n):
    """(A ⋈ B) ⋈ (C ⋈ D) on one variable: both inputs of the last join come
    out of a join already in key order (its sorts are skipped), small and
    semi-join-reduced sizes, with a repeated non-key column (equality mask);
    rows and order vs the oracle merge_join composed on the host."""
    rng = np.random.default_rng(n)
    hi = n // 6

    def tab(cols):
        return {c: rng.integers(1, hi if c == "x" else 50, size=n // 3).astype(np.uint32) for c in cols}

    A, B, C, D = tab(["x", "a"]), tab(["x", "b"]), tab(["x", "c"]), tab(["x", "a"])

    def host_join(L, R):
        pr = oq.merge_join(L["x"], R["x"]).reshape(-1, 2)
        out = {k: v[pr[:, 0]] for k, v in L.items()}
        keep = np.ones(len(pr), bool)
        for k, v in R.items():
            if k == "x":
                continue
            if k in out:
                keep &= out[k] == v[pr[:, 1]]
            else:
                out[k] = v[pr[:, 1]]
        return {k: v[keep] for k, v in out.items()}

    dev = {k: Q.DevTable.upload(list(t), t) for k, t in zip("ABCD", (A, B, C, D))}
    ab = Q._dev_join(dev["A"], dev["B"], "x", None)
    cd = Q._dev_join(dev["C"], dev["D"], "x", None)
    got = Q._dev_join(ab, cd, "x", None).download()
    want = host_join(host_join(A, B), host_join(C, D))
    assert got.columns == list(want)
    for c in got.columns:
        np.testing.assert_array_equal(got.data[c], want[c], err_msg=c)


def test_distinct_key_range_passes(gpu):
    """The first-occurrence table in several key-range passes (forced with a
    1 MB pass size in a fresh process): 1 and 2 columns vs the oracle."""
    import os
    import subprocess
    import sys
    code = """
import numpy as np, sys
sys.path[:0] = ['tests', '.']
from helpers import table_rows
from oracle import query as oq
from paper_1807_01409_b200 import query_ops as Q
rng = np.random.default_rng(5)
for cols, hi in ((['a'], 2**21), (['a', 'b'], 2**10)):
    data = {c: rng.integers(1, hi, size=400_000).astype(np.uint32) for c in cols}
    got = Q.project_distinct(Q.BindingTable(cols, data), cols, True)
    want = oq.project_distinct(oq.Table(cols, data), cols, True)
    np.testing.assert_array_equal(table_rows(got), want.rows())
print('OK')
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "TIDQ_DISTINCT_PASS_MB": "1"})
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("hot", [0, 5000])
def test_distinct_two_wide_columns_partition_and_hot_key(gpu, hot):
    """Two columns too wide for the first-occurrence table (hash-partition
    path), 1.2 M rows with duplicates; with `hot` copies of one row spread
    through the input its partition overflows the shared table and the
    DISTINCT falls back to the sort — same rows and order either way."""
    rng = np.random.default_rng(11 + hot)
    n = 1_200_000
    a = rng.integers(1, 2**31, size=n // 2, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(1, 2**31, size=n // 2, dtype=np.uint64).astype(np.uint32)
    idx = rng.integers(0, n // 2, size=n)  # every row about twice
    data = {"a": a[idx], "b": b[idx]}
    if hot:
        at = rng.choice(n, size=hot, replace=False)
        data["a"][at], data["b"][at] = 12345, 67890
    got = Q.project_distinct(Q.BindingTable(["a", "b"], data), ["a", "b"], True)
    want = oq.project_distinct(oq.Table(["a", "b"], data), ["a", "b"], True)
    np.testing.assert_array_equal(table_rows(got), want.rows())


@pytest.mark.parametrize("dups", ["rare", "many", "hot"])
def test_distinct_two_columns_5m(gpu, dups):
    """5 M-row two-column DISTINCT (the partition path): mostly-unique pairs
    (the C3 case), every pair ~3 times, and one pair 300 K times (partition
    overflow -> the sort) must all give numpy's first occurrences in order."""
    rng = np.random.default_rng({"rare": 1, "many": 2, "hot": 3}[dups])
    n = 5_000_000
    if dups == "many":
        m = n // 3
        a = rng.integers(1, 2**26, size=m, dtype=np.uint32)
        b = rng.integers(1, 2**26, size=m, dtype=np.uint32)
        idx = rng.integers(0, m, size=n)
        x, y = a[idx], b[idx]
    else:
        x = rng.integers(1, 2**26, size=n, dtype=np.uint32)
        y = rng.integers(1, 2**26, size=n, dtype=np.uint32)
        x[1::1000], y[1::1000] = x[::1000][: len(x[1::1000])], y[::1000][: len(y[1::1000])]  # some duplicates
        if dups == "hot":
            at = rng.choice(n, size=300_000, replace=False)
            x[at], y[at] = 7, 11
    data = {"x": x, "y": y}
    got = Q.project_distinct(Q.BindingTable(["x", "y"], data), ["x", "y"], True)
    key = (x.astype(np.uint64) << np.uint64(32)) | y
    _, first = np.unique(key, return_index=True)
    first.sort()
    np.testing.assert_array_equal(table_rows(got), np.stack([x[first], y[first]], axis=1))
