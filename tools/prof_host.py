"""Host-overhead probe: per-query wall time vs device time, cProfile of the
Python layer on the C2 sweep (run on the GPU box)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
from paper_1807_01409_b200 import _lib, plan, query_ops
from paper_1807_01409_b200.store import DeviceStore
from paper_1807_01409_b200.synth import SynthDictionary

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
ctx = _lib.context(0)
d = SynthDictionary(10_000, 10_000_000)
ds = DeviceStore.generate(n, seed=2, n_p=10_000, n_e=10_000_000)
qs = [plan.compile_query([plan.Group([plan.pattern("?s", f"<http://example.org/p/{r}>", "?o")], [])], d)
      for r in (1, 10, 100, 1000, 10000)]


def step():
    for q in qs:
        r = query_ops.evaluate_query_device(q, ds, d, row_cap=None)
        r.t.free()


for _ in range(3):
    step()
ctx.sync()
ctx.profile_reset()
ctx.profile(True)
t0 = time.perf_counter()
ctx.timer_begin()
for _ in range(10):
    step()
ms = ctx.timer_end()
wall = time.perf_counter() - t0
ctx.profile(False)
k_ms, k_n, _ = ctx.profile_read("scan")
print(f"per step: device {ms / 10:.3f} ms, wall {wall * 100:.3f} ms, scan kernels {k_ms / 10:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
