"""Host-side cost of the C2 sweep's evaluate_query_device calls (GPU box):
wall time per query with the GPU work queued asynchronously, and a cProfile
of the Python path."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_01409_b200 import _lib, plan, query_ops  # noqa: E402
from paper_1807_01409_b200.store import DeviceStore  # noqa: E402
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary  # noqa: E402

c = CONFIGS["C2"]
ds = DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"])
d = SynthDictionary(c["n_p"], c["n_e"])
qs = [plan.compile_query([plan.Group([plan.pattern("?s", f"<http://example.org/p/{r}>", "?o")], [])], d)
      for r in (1, 10, 100, 1000, 10000)]
ctx = _lib.context()


def step(collect=True):
    res = [query_ops.evaluate_query_device(q, ds, d, row_cap=None) for q in qs]
    t_launch = time.perf_counter()
    for r in res:
        r.n_rows
        r.t.free()
    return t_launch


for _ in range(5):
    step()
ctx.sync()
N = 50
host = 0.0
t0 = time.perf_counter()
for _ in range(N):
    a = time.perf_counter()
    b = step()
    host += b - a
wall = (time.perf_counter() - t0) / N
print(f"step wall {wall * 1e3:.3f} ms; host launch part {host / N * 1e3:.3f} ms per step "
      f"({host / N / 5 * 1e6:.1f} us per query)")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
