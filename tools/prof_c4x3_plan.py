import cProfile, pstats, os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tools'))
import bench_configs as bc
from paper_1807_01409_b200 import _lib, query_ops
from paper_1807_01409_b200.store import DeviceStore
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary
c = CONFIGS["C4"]
ds = DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"]).prepare()
d = SynthDictionary(c["n_p"], c["n_e"])
q = bc.q_star(d, [3, 5, 7], None)
ctx = _lib.context()
for _ in range(5): query_ops.evaluate_query_device(q, ds, d).n_rows
ctx.sync()
# time only the planning part: _scan_device up to run_scan (patch run_scan to record time)
real_run = _lib.run_scan
marks = []
def rs(*a, **k):
    marks.append(time.perf_counter())
    return real_run(*a, **k)
_lib.run_scan = rs
query_ops._lib.run_scan = rs
N = 50; pre = 0.0
for _ in range(N):
    ctx.sync(); marks.clear()
    t = time.perf_counter()
    r = query_ops.evaluate_query_device(q, ds, d)
    pre += marks[0] - t
    r.n_rows
print(f"host time from call to run_scan: {pre / N * 1e6:.1f} us")
pr = cProfile.Profile(); pr.enable()
for _ in range(N):
    query_ops.evaluate_query_device(q, ds, d).n_rows
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(18)
