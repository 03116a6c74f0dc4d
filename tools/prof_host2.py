"""Per-query host timeline: wall time of the ctypes scan call vs the Python
layer around it (run on the GPU box)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1807_01409_b200 import _lib, plan, query_ops
from paper_1807_01409_b200.store import DeviceStore
from paper_1807_01409_b200.synth import SynthDictionary

ctx = _lib.context(0)
d = SynthDictionary(10_000, 10_000_000)
ds = DeviceStore.generate(100_000_000, seed=2, n_p=10_000, n_e=10_000_000)
qs = [plan.compile_query([plan.Group([plan.pattern("?s", f"<http://example.org/p/{r}>", "?o")], [])], d)
      for r in (1, 10, 100, 1000, 10000)]
orig = _lib.run_scan
acc = {"scan": 0.0}


def timed(*a, **k):
    t = time.perf_counter()
    r = orig(*a, **k)
    acc["scan"] += time.perf_counter() - t
    return r


query_ops._lib.run_scan = timed
for q in qs:
    query_ops.evaluate_query_device(q, ds, d, row_cap=None).t.free()
for rep in range(3):
    acc["scan"] = 0.0
    t0 = time.perf_counter()
    for _ in range(20):
        for q in qs:
            r = query_ops.evaluate_query_device(q, ds, d, row_cap=None)
            r.t.free()
    wall = time.perf_counter() - t0
    print(f"per query: wall {wall / 100 * 1e6:.1f} us, inside run_scan {acc['scan'] / 100 * 1e6:.1f} us")
t = time.perf_counter()
for _ in range(1000):
    ctx.launches
print(f"one trivial ctypes call: {(time.perf_counter() - t) * 1e3:.2f} us")
