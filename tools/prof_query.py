"""Run one C3/C4 query a few times (for ncu launch lists)."""
import sys

sys.path.insert(0, ".")
from paper_1807_01409_b200 import _lib, plan, query_ops
from paper_1807_01409_b200.store import DeviceStore
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary

which = sys.argv[1] if len(sys.argv) > 1 else "distinct"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = CONFIGS["C3"]
ds = DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"])
d = SynthDictionary(c["n_p"], c["n_e"])
P = "<http://example.org/p/{}>"
if which == "distinct":
    q = plan.compile_query([plan.Group([plan.pattern("?s", P.format(r), "?o")], []) for r in (2, 3, 4, 5)], d,
                           distinct=True, projection=["s"])
elif which == "distinct2":
    q = plan.compile_query([plan.Group([plan.pattern("?s", P.format(r), "?o")], []) for r in (2, 3, 4, 5)], d,
                           distinct=True, projection=["s", "o"])
else:
    q = plan.compile_query([plan.Group([plan.pattern("?s", P.format(3), "?o1"),
                                        plan.pattern("?s", P.format(5), "?o2")], [])], d)
for _ in range(reps):
    r = query_ops.evaluate_query_device(q, ds, d, row_cap=None)
    r.t.free()
_lib.context().sync()
