import cProfile, pstats, os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1807_01409_b200 import _lib, plan, query_ops
from paper_1807_01409_b200.store import DeviceStore
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary
c = CONFIGS["C2"]
ds = DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"]).prepare()
d = SynthDictionary(c["n_p"], c["n_e"])
qs = [plan.compile_query([plan.Group([plan.pattern("?s", f"<http://example.org/p/{r}>", "?o")], [])], d) for r in (1, 10, 100, 1000, 10000)]
ctx = _lib.context()
def q1():
    r = query_ops.evaluate_query_device(qs[4], ds, d, row_cap=None)
    ctx.sync()
    r.t.free()
for _ in range(50): q1()
# wall per query with sync excluded
tt=0
for _ in range(300):
    ctx.sync(); t=time.perf_counter(); r = query_ops.evaluate_query_device(qs[4], ds, d, row_cap=None); tt+=time.perf_counter()-t; ctx.sync(); r.t.free()
print("host per query (rank 10000)", tt/300*1e6, "us")
pr = cProfile.Profile(); pr.enable()
for _ in range(300):
    r = query_ops.evaluate_query_device(qs[4], ds, d, row_cap=None); ctx.sync(); r.t.free()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
