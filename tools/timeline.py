"""Warm GPU timeline of one BASELINE config query (run on the GPU box): the
query runs a few times under torch.profiler (CUPTI kernel activity — no
replay, no cache flush), and the last run's kernels are listed with the idle
gaps between them, so host-side waits (row-count syncs, launch latency) show
up next to the kernel time.

    python tools/timeline.py C4 "star x3" [reps] [nocap]

(the reference's default row cap unless "nocap": row_cap=None)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1807_01409_b200 import _lib, query_ops  # noqa: E402
from paper_1807_01409_b200.store import DeviceStore  # noqa: E402
from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary  # noqa: E402
import bench_configs as bc  # noqa: E402

cfg, name = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ROW_CAP = None if len(sys.argv) > 4 and sys.argv[4] == "nocap" else query_ops.DEFAULT_ROW_CAP
c = CONFIGS[cfg]
ds = DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"]).prepare()
d = SynthDictionary(c["n_p"], c["n_e"])
flt = "7$" if "FILTER" in name else None
k = int(name.split("x")[1].split()[0]) if " x" in name else 0
qs = None
if cfg == "C2":  # the bench sweep: "sweep" = all five ranks, "rank R" = one query
    ranks = [1, 10, 100, 1000, 10000] if name == "sweep" else [int(name.split()[1])]
    qs = [bc.plan.compile_query([bc.plan.Group([bc.plan.pattern("?s", bc.P.format(r), "?o")], [])], d)
          for r in ranks]
    q = qs[0]
elif cfg == "C3":
    ranks = list(range(2, 2 + k))
    if "bag" in name:
        q = bc.plan.compile_query([bc.plan.Group([bc.plan.pattern("?s", bc.P.format(r), "?o")], [])
                                   for r in ranks], d)
    else:
        q = bc.q_union(d, ranks, ["s", "o"] if "?o" in name else ["s"])
else:
    ranks = [3, 5, 7, 11][:k] if cfg == "C4" else [5, 7, 11]
    q = bc.q_star(d, ranks, flt) if "star" in name else bc.q_chain(d, ranks, flt)
ctx = _lib.context()
qs = qs or [q]


def run_once():
    res = [query_ops.evaluate_query_device(x, ds, d, row_cap=ROW_CAP) for x in qs]
    for r in res:
        r.n_rows
        r.t.free()


for _ in range(2):
    run_once()
ctx.sync()
torch.cuda.synchronize()
marker = torch.empty(1, device="cuda")
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(reps):
        ctx.sync()
        marker.fill_(1)  # run delimiter on the timeline
        torch.cuda.synchronize()
        run_once()
        ctx.sync()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev], key=lambda x: x[0])
# split into queries at the delimiter kernels
runs, cur = [], []
for k_ in kern:
    if "fill" in k_[2].lower() and "tidq" not in k_[2]:
        if cur:
            runs.append(cur)
        cur = []
        continue
    cur.append(k_)
runs.append(cur)
last = runs[-1]
t0 = last[0][0]
busy = sum(b - a for a, b, _ in last)
span = last[-1][1] - t0
print(f"{cfg} {name}: {len(runs)} runs, last run: span {span:.1f} us, kernels busy {busy:.1f} us, "
      f"idle {span - busy:.1f} us, {len(last)} kernels/copies")
prev_end = t0
for a, b, nm in last:
    gap = a - prev_end
    print(f"  +{a - t0:8.1f}  gap {gap:7.1f}  dur {b - a:8.1f}  {nm[:80]}")
    prev_end = max(prev_end, b)
