"""Breakdown of bench.py's e2e step on the GPU box: store upload from pinned
memory, the 5 queries on the device, and the result downloads."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1807_01409_b200 import _lib, query_ops  # noqa: E402
from paper_1807_01409_b200.store import DeviceStore, TripleChunk  # noqa: E402
from paper_1807_01409_b200.synth import SynthDictionary  # noqa: E402

n = bench.N_TRIPLES
ctx = _lib.context(0)
d = SynthDictionary(bench.N_P, n // 10)
qs = bench.queries(d)
ds = DeviceStore.generate(n, seed=bench.SEED, n_p=bench.N_P, n_e=n // 10)
p = ctypes.c_void_p()
_lib.call("tidq_host_alloc", n * 12, ctypes.byref(p))
host = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint32)), shape=(n * 3,))
host[:] = ds.download().reshape(-1)
ds.free()
chunk = TripleChunk(host, 0)
acc = {"upload": 0.0, "device": 0.0, "download": 0.0, "free": 0.0}
for rep in range(4):
    t0 = time.perf_counter()
    st = DeviceStore.upload(chunk)
    t1 = time.perf_counter()
    res = [query_ops.evaluate_query_device(q, st, d, row_cap=None) for q in qs]
    ctx.sync()
    t2 = time.perf_counter()
    tabs = [r.download() for r in res]
    t3 = time.perf_counter()
    for r in res:
        r.t.free()
    st.free()
    t4 = time.perf_counter()
    if rep:
        for k, v in zip(acc, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
            acc[k] += v / 3
nbytes = sum(t.data[c].nbytes for t in tabs for c in t.columns)
print({k: round(v * 1e3, 2) for k, v in acc.items()}, "ms;", nbytes / 1e6, "MB downloaded",
      f"({nbytes / acc['download'] / 1e9:.1f} GB/s)")
