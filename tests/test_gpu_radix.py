"""The device radix sort (onesweep and the three-kernel LSD passes, env
TIDQ_RADIX) against numpy's stable argsort: every join, DISTINCT and
partition on the query path sorts through it, and the reference's row order
(merge_join's stable argsorts, query_ops.py:110-118,163-166) depends on its
stability."""

import numpy as np
import pytest

from paper_1807_01409_b200._sortdiag import radix_sort

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["onesweep", "lsd"])
def impl(request, monkeypatch):
    monkeypatch.setenv("TIDQ_RADIX", request.param)
    return request.param


def _check(keys, bits):
    vals = np.arange(len(keys), dtype=np.uint32)
    sk, sv, _ = radix_sort(keys, vals, bits)
    mask = np.array((1 << bits) - 1 if bits < 8 * keys.itemsize else -1, dtype=np.int64).astype(keys.dtype)
    order = np.argsort(keys & mask, kind="stable")
    assert np.array_equal(sv, order.astype(np.uint32))
    assert np.array_equal(sk, keys[order])


@pytest.mark.parametrize("n", [1, 2, 31, 4095, 4096, 4097, 100_003, 2_000_000])
@pytest.mark.parametrize("bits", [1, 8, 13, 28, 32])
def test_radix_u32_uniform(gpu, impl, n, bits):
    rng = np.random.default_rng(n * 131 + bits)
    keys = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    if bits < 32:
        keys &= np.uint32((1 << bits) - 1)
    _check(keys, bits)


@pytest.mark.parametrize("kind", ["equal", "few", "sorted", "reversed", "high_only", "skew"])
def test_radix_u32_distributions(gpu, impl, kind):
    n = 1_500_017
    rng = np.random.default_rng(7)
    if kind == "equal":
        keys = np.full(n, 12345, dtype=np.uint32)
    elif kind == "few":
        keys = rng.choice(np.array([3, 70000, 2**27 + 5], dtype=np.uint32), n)
    elif kind == "sorted":
        keys = np.sort(rng.integers(0, 2**28, n, dtype=np.uint32))
    elif kind == "reversed":
        keys = np.sort(rng.integers(0, 2**28, n, dtype=np.uint32))[::-1].copy()
    elif kind == "high_only":
        keys = (rng.integers(0, 16, n, dtype=np.uint32) << np.uint32(24))
    else:  # one hot key in most rows
        keys = rng.integers(0, 2**28, n, dtype=np.uint32)
        keys[rng.random(n) < 0.9] = 2**20 + 3
    _check(keys, 28 if kind != "equal" else 14)


def test_radix_u32_above_2p24(gpu, impl):
    # the LSD path switches to 9-10-bit digits above 2^24 keys
    rng = np.random.default_rng(11)
    keys = rng.integers(0, 2**28, 20_000_000, dtype=np.uint32)
    _check(keys, 28)


@pytest.mark.parametrize("n,bits", [(3, 64), (4097, 16), (1_000_003, 16), (1_000_003, 40), (300_001, 64)])
def test_radix_u64(gpu, impl, n, bits):
    rng = np.random.default_rng(bits + n)
    keys = rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    if bits < 64:
        keys &= np.uint64((1 << bits) - 1)
    keys[::7] = keys[min(3, n - 1)]  # duplicates: stability
    _check(keys, bits)

