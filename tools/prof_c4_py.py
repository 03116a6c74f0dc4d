"""Host-side (Python) profile of one C4 star x2 query on the GPU box: wall
time of evaluate_query_device with the GPU idle before it, and a cProfile."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench_configs as bc  # noqa: E402
from paper_1807_01409_b200 import _lib, query_ops  # noqa: E402
from paper_1807_01409_b200.store import DeviceStore  # noqa: E402
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary  # noqa: E402

c = CONFIGS["C4"]
ds = DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"]).prepare()
d = SynthDictionary(c["n_p"], c["n_e"])
q = bc.q_star(d, [3, 5], None)
ctx = _lib.context()
for _ in range(5):
    query_ops.evaluate_query_device(q, ds, d).n_rows
ctx.sync()
N = 30
tt = 0.0
for _ in range(N):
    ctx.sync()
    t = time.perf_counter()
    r = query_ops.evaluate_query_device(q, ds, d)
    r.n_rows
    tt += time.perf_counter() - t
print(f"C4 star x2 wall per query {tt / N * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    query_ops.evaluate_query_device(q, ds, d).n_rows
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
