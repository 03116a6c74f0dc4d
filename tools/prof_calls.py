"""Wall time per libtidq ABI call for one BASELINE config query (run on the
GPU box): every ABI call is synchronous, so this is the query's device+host
timeline by operator.

    python tools/prof_calls.py C4 "star x2" [reps]
"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1807_01409_b200 import _lib, query_ops  # noqa: E402
from paper_1807_01409_b200.store import DeviceStore  # noqa: E402
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary  # noqa: E402
import bench_configs as bc  # noqa: E402

cfg, name = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
c = CONFIGS[cfg]
ds = DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"])
d = SynthDictionary(c["n_p"], c["n_e"])
flt = "7$" if "FILTER" in name else None
k = int(name.split("x")[1].split()[0])
if cfg == "C3":
    ranks = list(range(2, 2 + k))
    if "bag" in name:
        q = bc.plan.compile_query([bc.plan.Group([bc.plan.pattern("?s", bc.P.format(r), "?o")], [])
                                   for r in ranks], d)
    else:
        q = bc.q_union(d, ranks, ["s", "o"] if "?o" in name else ["s"])
else:
    ranks = [3, 5, 7, 11][:k] if cfg == "C4" else [5, 7, 11]
    q = bc.q_star(d, ranks, flt) if "star" in name else bc.q_chain(d, ranks, flt)
acc = collections.defaultdict(lambda: [0.0, 0])
orig = _lib.call


def timed(fn, *a):
    t = time.perf_counter()
    r = orig(fn, *a)
    e = acc[fn]
    e[0] += time.perf_counter() - t
    e[1] += 1
    return r


_lib.call = timed
query_ops._lib.call = timed
r = query_ops.evaluate_query_device(q, ds, d, row_cap=None)
r.t.free()
acc.clear()
ctx = _lib.context()
ctx.sync()
t0 = time.perf_counter()
for _ in range(reps):
    r = query_ops.evaluate_query_device(q, ds, d, row_cap=None)
    rows = r.n_rows
    r.t.free()
wall = (time.perf_counter() - t0) / reps * 1e3
print(f"{cfg} {name}: {rows} rows, {wall:.3f} ms per query (wall)")
ctx.profile_reset()
ctx.profile(True)
for _ in range(reps):
    query_ops.evaluate_query_device(q, ds, d, row_cap=None).t.free()
ctx.profile(False)
for kname in ("scan.mark", "scan"):
    ms, n, b = ctx.profile_read(kname)
    if n:
        print(f"  [events] {kname:10s} {ms / reps:8.3f} ms/query  {b / (ms / 1e3) / 1e9 if ms else 0:8.1f} GB/s algorithmic")
for fn, (t, n) in sorted(acc.items(), key=lambda x: -x[1][0]):
    print(f"  {fn:28s} {t / reps * 1e3:8.3f} ms  x{n // reps}")
