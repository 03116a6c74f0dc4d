"""Latency of the BASELINE.json configs C3 (UNION + DISTINCT), C4 (star/chain
joins with FILTER) and C5 (2B-triple 3-way joins) on one B200, plus
size-independent property checks of the results.  Writes one JSON line per
query to stdout.

    python tools/bench_configs.py [--configs C3,C4] [--scale 1.0] [--reps 3]
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

from paper_1807_01409_b200 import _lib, plan, query_ops  # noqa: E402
from paper_1807_01409_b200.store import DeviceStore  # noqa: E402
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary  # noqa: E402

P = "<http://example.org/p/{}>"


def q_union(d, ranks, distinct_vars):
    groups = [plan.Group([plan.pattern("?s", P.format(r), "?o")], []) for r in ranks]
    return plan.compile_query(groups, d, distinct=True, projection=distinct_vars)


def q_star(d, ranks, flt=None):
    pats = [plan.pattern("?s", P.format(r), f"?o{i + 1}") for i, r in enumerate(ranks)]
    filters = [plan.Filter("o1", flt)] if flt else []
    return plan.compile_query([plan.Group(pats, filters)], d)


def q_chain(d, ranks, flt=None):
    names = ["x", "y", "z", "w", "v"]
    pats = [plan.pattern(f"?{names[i]}", P.format(r), f"?{names[i + 1]}") for i, r in enumerate(ranks)]
    filters = [plan.Filter("y", flt)] if flt else []
    return plan.compile_query([plan.Group(pats, filters)], d)


ONLY = None
ROW_CAP = query_ops.DEFAULT_ROW_CAP


def run(name, q, ds, d, reps, ctx, check=None):
    if ONLY and ONLY not in name:
        return None
    res = query_ops.evaluate_query_device(q, ds, d, row_cap=ROW_CAP)  # warm (filter cache, pools)
    n = res.n_rows
    res.t and res.t.free()
    times = []
    for _ in range(reps):
        ctx.sync()
        ctx.timer_begin()
        t0 = time.perf_counter()
        res = query_ops.evaluate_query_device(q, ds, d, row_cap=ROW_CAP)
        dev = ctx.timer_end()
        times.append((dev, (time.perf_counter() - t0) * 1e3))
        if _ is not reps - 1:
            res.t and res.t.free()
    rec = {"query": name, "rows": n, "device_ms": min(t[0] for t in times),
           "wall_ms": min(t[1] for t in times), "reps": reps}
    if check is not None:
        rec["check"] = check(res)
    res.t and res.t.free()
    print(json.dumps(rec), flush=True)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C3,C4")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--only", default=None, help="run only queries whose name contains this")
    ap.add_argument("--nocap", action="store_true", help="row_cap=None (semi-join-reduced star path)")
    a = ap.parse_args()
    global ONLY, ROW_CAP
    ONLY = a.only
    if a.nocap:
        ROW_CAP = None
    ctx = _lib.context(0)
    for cfg in a.configs.split(","):
        c = dict(CONFIGS[cfg])
        n = int(c["n_triples"] * a.scale)
        n_e = max(1, int(c["n_e"] * a.scale))
        t0 = time.perf_counter()
        ds = DeviceStore.generate(n, seed=c["seed"], n_p=c["n_p"], n_e=n_e)
        d = SynthDictionary(c["n_p"], n_e)
        print(json.dumps({"config": cfg, "triples": n, "n_e": n_e,
                          "generate_s": round(time.perf_counter() - t0, 3)}), flush=True)
        ds.prepare()  # index columns at load time (as bench.py)
        hist = ds.predicate_counts()
        if cfg == "C3":
            for k in (4, 8):
                ranks = list(range(2, 2 + k))
                run(f"C3 DISTINCT ?s UNION x{k}", q_union(d, ranks, ["s"]), ds, d, a.reps, ctx)
                run(f"C3 DISTINCT ?s ?o UNION x{k}", q_union(d, ranks, ["s", "o"]), ds, d, a.reps, ctx)
                run(f"C3 UNION x{k} (bag)", plan.compile_query(
                    [plan.Group([plan.pattern("?s", P.format(r), "?o")], []) for r in ranks], d),
                    ds, d, a.reps, ctx,
                    check=lambda res, ranks=ranks: bool(res.n_rows == int(sum(hist[r] for r in ranks))))
        if cfg in ("C4",):
            for k in (2, 3, 4):
                ranks = [3, 5, 7, 11][:k]
                run(f"C4 star x{k}", q_star(d, ranks), ds, d, a.reps, ctx)
                run(f"C4 star x{k} FILTER", q_star(d, ranks, "7$"), ds, d, a.reps, ctx)
                run(f"C4 chain x{k}", q_chain(d, ranks), ds, d, a.reps, ctx)
                run(f"C4 chain x{k} FILTER", q_chain(d, ranks, "7$"), ds, d, a.reps, ctx)
        if cfg == "C5":
            run("C5 star x3", q_star(d, [5, 7, 11]), ds, d, a.reps, ctx)
            run("C5 chain x3", q_chain(d, [5, 7, 11]), ds, d, a.reps, ctx)
        ds.free()


if __name__ == "__main__":
    main()
