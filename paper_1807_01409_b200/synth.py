"""Synthetic TripleID data: Zipf CDF table and dictionary shim.

The device generator (csrc/store.cu ``generate_kernel``) draws triple i as
    h_j = splitmix64(((i << 2) | j) ^ (seed * 0xD1B54A32D192ED03))
    p   = 1 + first r with h_1 < T[r]                 (Zipf(s) over n_p predicates)
    s   = n_p + 1 + (((h_0 >> 32) * n_e) >> 32)      (shared entity pool, so
    o   = n_p + 1 + (((h_2 >> 32) * n_e) >> 32)       OS/SO chains are non-empty)
``T`` is computed here once and handed to the device, so device data and the
oracle's numpy twin (oracle/synth.py) are bit-identical.

The reference's ``datagen.py`` is unusable for the BASELINE configs (uniform
predicates, disjoint s/o namespaces, text path); see SURVEY §2.
"""

from __future__ import annotations

import numpy as np

__all__ = ["zipf_cdf_table", "SynthDictionary", "CONFIGS", "predicate_id", "expected_fraction"]


def zipf_cdf_table(n_p: int, s: float = 1.0) -> np.ndarray:
    """uint64 T[r] = floor(CDF(r) * 2^64), T[n_p-1] = 2^64 - 1."""
    ranks = np.arange(1, n_p + 1, dtype=np.float64)
    w = ranks ** (-float(s))
    cdf = np.cumsum(w) / w.sum()
    t = np.empty(n_p, dtype=np.uint64)
    scaled = cdf[:-1] * 18446744073709551616.0
    # values < 2^64 convert exactly; guard the rounding edge
    scaled = np.minimum(scaled, 18446744073709549568.0)
    t[:-1] = scaled.astype(np.uint64)
    t[-1] = np.uint64(0xFFFFFFFFFFFFFFFF)
    return t


def predicate_id(rank: int) -> int:
    """ID of the predicate of Zipf rank ``rank`` (1-based)."""
    return int(rank)


def expected_fraction(rank: int, n_p: int = 10_000, s: float = 1.0) -> float:
    h = float(np.sum(np.arange(1, n_p + 1, dtype=np.float64) ** (-s)))
    return rank ** (-s) / h


class SynthDictionary:
    """Duck-typed stand-in for ``tripleid.dictionary.Dictionary`` over the
    generator's ID space: predicates ``<http://example.org/p/{id}>`` for
    1..n_p, entities ``<http://example.org/e/{k}>`` for id = n_p + k."""

    def __init__(self, n_p: int, n_e: int):
        self.n_p = int(n_p)
        self.n_e = int(n_e)

    def __len__(self) -> int:
        return self.n_p + self.n_e

    @property
    def max_id(self) -> int:
        return self.n_p + self.n_e

    def decode_lexical(self, ident: int) -> str:
        ident = int(ident)
        if ident <= 0 or ident > self.max_id:
            raise KeyError(ident)
        if ident <= self.n_p:
            return f"<http://example.org/p/{ident}>"
        return f"<http://example.org/e/{ident - self.n_p}>"

    def lookup(self, lexical: str) -> int | None:
        for prefix, off, hi in (("<http://example.org/p/", 0, self.n_p),
                                ("<http://example.org/e/", self.n_p, self.n_e)):
            if lexical.startswith(prefix) and lexical.endswith(">"):
                body = lexical[len(prefix):-1]
                if body.isdigit():
                    k = int(body)
                    if 1 <= k <= hi:
                        return k + off
        return None


# BASELINE.json configs as concrete synthetic stores
CONFIGS = {
    "C1": dict(n_triples=1_000_000, seed=1, n_p=10_000, n_e=100_000),
    "C2": dict(n_triples=100_000_000, seed=2, n_p=10_000, n_e=10_000_000),
    "C3": dict(n_triples=500_000_000, seed=3, n_p=10_000, n_e=50_000_000),
    "C4": dict(n_triples=500_000_000, seed=3, n_p=10_000, n_e=50_000_000),
    "C5": dict(n_triples=2_000_000_000, seed=5, n_p=10_000, n_e=200_000_000),
}
