"""numpy twin of the device generator — TEST INFRASTRUCTURE.

Bit-identical to csrc/store.cu ``generate_kernel`` given the same Zipf CDF
table (``paper_1807_01409_b200.synth.zipf_cdf_table`` — a host-side table the
product hands to the device).  Used to build the oracle's AoS chunks for
parity and for the CPU baseline.
"""

from __future__ import annotations

import numpy as np

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def generate(n_triples: int, *, seed: int, n_p: int, n_e: int, cdf: np.ndarray,
             base_index: int = 0, block: int = 1 << 22, threads: int = 1) -> np.ndarray:
    """(n_triples, 3) uint32 rows of triples base_index .. base_index+n-1.
    ``threads`` > 1 fills blocks concurrently (numpy releases the GIL in the
    hashing ufuncs and searchsorted); the rows are identical."""
    out = np.empty((n_triples, 3), dtype=np.uint32)
    with np.errstate(over="ignore"):
        salt = np.uint64(seed) * np.uint64(0xD1B54A32D192ED03)
    ent0 = np.uint64(n_p + 1)

    def fill(lo):
        hi = min(n_triples, lo + block)
        g = (np.arange(base_index + lo, base_index + hi, dtype=np.uint64) << np.uint64(2))
        h0 = splitmix64(g ^ salt)
        h1 = splitmix64((g | np.uint64(1)) ^ salt)
        h2 = splitmix64((g | np.uint64(2)) ^ salt)
        r = np.searchsorted(cdf, h1, side="right")
        np.minimum(r, n_p - 1, out=r)
        out[lo:hi, 1] = (r + 1).astype(np.uint32)
        with np.errstate(over="ignore"):
            out[lo:hi, 0] = (ent0 + (((h0 >> np.uint64(32)) * np.uint64(n_e)) >> np.uint64(32))).astype(np.uint32)
            out[lo:hi, 2] = (ent0 + (((h2 >> np.uint64(32)) * np.uint64(n_e)) >> np.uint64(32))).astype(np.uint32)

    starts = range(0, n_triples, block)
    if threads > 1 and n_triples > block:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(fill, starts))
    else:
        for lo in starts:
            fill(lo)
    return out
