"""Host-side breakdown of one C2 sweep query on the GPU box: wall time of
every libtidq C call the Python path makes (per name, per query), and the
tidq_scan phases (TIDQ_HOST_TRACE)."""
import collections
import os
import sys
import time

os.environ.setdefault("TIDQ_HOST_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_01409_b200 import _lib, plan, query_ops  # noqa: E402
from paper_1807_01409_b200.store import DeviceStore  # noqa: E402
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary  # noqa: E402

c = CONFIGS["C2"]
ds = DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"]).prepare()
d = SynthDictionary(c["n_p"], c["n_e"])
qs = [plan.compile_query([plan.Group([plan.pattern("?s", f"<http://example.org/p/{r}>", "?o")], [])], d)
      for r in (1, 10, 100, 1000, 10000)]
ctx = _lib.context()
stat = collections.defaultdict(lambda: [0, 0.0])
real = _lib.call


def timed(name, *args):
    t = time.perf_counter()
    try:
        return real(name, *args)
    finally:
        s = stat[name]
        s[0] += 1
        s[1] += time.perf_counter() - t


def step():
    res = [query_ops.evaluate_query_device(q, ds, d, row_cap=None) for q in qs]
    for r in res:
        r.n_rows
        r.t.free()


for _ in range(10):
    step()
ctx.sync()
_lib.call = timed
query_ops._lib.call = timed
N = 100
t_first = 0.0
for _ in range(N):
    ctx.sync()
    t = time.perf_counter()
    r = query_ops.evaluate_query_device(qs[0], ds, d, row_cap=None)
    t_first += time.perf_counter() - t
    r.n_rows
    r.t.free()
    step()
print(f"first query of a step, host: {t_first / N * 1e6:.1f} us")
for k, (n, s) in sorted(stat.items(), key=lambda x: -x[1][1]):
    print(f"{k:32s} calls/query {n / (N * 6):5.2f}  us/call {s / n * 1e6:7.1f}")
