"""Entailment (§8f row 2) latency: device run_rule on a resident RDFS-shaped
store, split into the two device searches and the host tables/conclusions
the reference API returns.  One JSON line per rule.  (The CPU reference
algorithm is timed by tests only: tools never run oracle/.)

    python tools/bench_entail.py [--triples 2000000]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import VocabDictionary  # noqa: E402
from test_gpu_entail import _big_store  # noqa: E402

from paper_1807_01409_b200 import _lib  # noqa: E402
from paper_1807_01409_b200 import entailment as E  # noqa: E402
from paper_1807_01409_b200.store import DeviceStore, TripleChunk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--triples", type=int, default=2_000_000)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    ctx = _lib.context(0)
    rows, vocab, max_id = _big_store(7, a.triples)
    ds = DeviceStore.upload(TripleChunk(rows.reshape(-1), 0))
    for rule in sorted(E.RULES):
        E.run_rule(rule, ds, VocabDictionary(max_id, vocab))
        ts, tm = [], {}
        for _ in range(a.reps):
            ctx.sync()
            t = time.perf_counter()
            run = E.run_rule(rule, ds, VocabDictionary(max_id, vocab), timings=tm)
            ts.append(time.perf_counter() - t)
        print(json.dumps({"rule": rule, "triples": a.triples, "gpu_ms": round(min(ts) * 1e3, 3),
                          "gpu_search_ms": round(tm["search"] * 1e3, 3),
                          "host_tables_ms": round(tm["tables"] * 1e3, 3),
                          "gpu_triples_per_s": a.triples / min(ts),
                          "counts": list(E.report_counts(run)),
                          "stage2_links": len(run.stage1_table)}), flush=True)


if __name__ == "__main__":
    main()
