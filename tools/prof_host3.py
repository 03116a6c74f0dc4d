import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
from paper_1807_01409_b200 import _lib, query_ops
from paper_1807_01409_b200.store import DeviceStore
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary
import bench_configs as bc
c = CONFIGS["C4"]
ds = DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"])
d = SynthDictionary(c["n_p"], c["n_e"])
q = bc.q_star(d, [3, 5])
for _ in range(3):
    r = query_ops.evaluate_query_device(q, ds, d, row_cap=None); r.n_rows; r.t.free()
ctx = _lib.context(); ctx.sync()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(50):
    r = query_ops.evaluate_query_device(q, ds, d, row_cap=None); r.n_rows; r.t.free()
pr.disable()
print("wall per query ms", (time.perf_counter() - t0) / 50 * 1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
