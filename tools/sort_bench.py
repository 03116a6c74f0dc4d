"""A/B timing of the device radix sort implementations (TIDQ_RADIX) on the
sizes the query path sorts: join sides (28-bit term-ID keys), the DISTINCT
partition sort (64-bit keys by their low 16 bits).  One JSON line per case.

    python tools/sort_bench.py [--impl onesweep,lsd] [--reps 10]
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1807_01409_b200._sortdiag import radix_sort  # noqa: E402

CASES = [  # (name, n, key bytes, bits)
    ("join 0.5M x28", 500_000, 4, 28),
    ("join 3.4M x28 (C4)", 3_400_000, 4, 28),
    ("join 5.5M x28 (C5)", 5_500_000, 4, 28),
    ("join 20M x28", 20_000_000, 4, 28),
    ("partition 65M u64 x16 (C3 x4)", 65_000_000, 8, 16),
    ("partition 93M u64 x16 (C3 x8)", 93_000_000, 8, 16),
    ("sort 10M u64 x52", 10_000_000, 8, 52),
]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", default="onesweep,lsd")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="", help="substring of the case names to run")
    a = ap.parse_args()
    rng = np.random.default_rng(1)
    for name, n, kb, bits in CASES:
        if a.only not in name:
            continue
        if kb == 4:
            keys = rng.integers(0, 1 << bits, n, dtype=np.uint32)
        else:
            keys = rng.integers(0, 2**63, n, dtype=np.uint64) & np.uint64((1 << bits) - 1)
        vals = np.arange(n, dtype=np.uint32)
        want = None
        for impl in a.impl.split(","):
            os.environ["TIDQ_RADIX"] = impl
            sk, sv, ms = radix_sort(keys, vals, bits, reps=a.reps)
            if want is None:
                mask = (1 << bits) - 1
                want = np.argsort(keys & keys.dtype.type(mask), kind="stable").astype(np.uint32)
            ok = bool(np.array_equal(sv, want))
            passes = -(-bits // 8)
            gbs = n * (kb + 4) * 2 * passes / (ms * 1e-3) / 1e9 if ms else 0.0
            print(json.dumps({"case": name, "impl": impl, "n": n, "key_bytes": kb, "bits": bits, "ms": round(ms, 4),
                              "gkeys_s": round(n / (ms * 1e-3) / 1e9, 2), "pass_traffic_gbs_8bit": round(gbs, 1),
                              "stable_ok": ok}), flush=True)


if __name__ == "__main__":
    main()
