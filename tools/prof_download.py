"""Download-path micro-benchmark (GPU box): D2H of a 40 MB column into fresh,
pre-touched and pinned host memory."""
import ctypes, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1807_01409_b200 import _lib
from paper_1807_01409_b200.query_ops import DevTable
ctx = _lib.context(0)
n = 10_000_000
t = DevTable.upload(["a"], {"a": np.arange(n, dtype=np.uint32)})
def tm(f, reps=5):
    f(); t0 = time.perf_counter()
    for _ in range(reps): f()
    return (time.perf_counter() - t0) / reps
pre = np.empty(n, np.uint32); pre[:] = 1
def fresh():
    a = np.empty(n, np.uint32)
    _lib.call("tidq_table_download_col", t.t.handle, 0, a.ctypes.data)
print("fresh np.empty   %.2f GB/s" % (n*4 / tm(fresh) / 1e9))
print("pre-touched      %.2f GB/s" % (n*4 / tm(lambda: _lib.call("tidq_table_download_col", t.t.handle, 0, pre.ctypes.data)) / 1e9))
keep = []
def pin():
    a = _lib.pinned_empty(n, np.uint32); _lib.call("tidq_table_download_col", t.t.handle, 0, a.ctypes.data)
print("pinned pool      %.2f GB/s" % (n*4 / tm(pin) / 1e9))
def pin_keep():
    a = _lib.pinned_empty(n, np.uint32); keep.append(a); _lib.call("tidq_table_download_col", t.t.handle, 0, a.ctypes.data)
print("pinned new alloc %.2f GB/s" % (n*4 / tm(pin_keep) / 1e9))
print("column()         %.2f GB/s" % (n*4 / tm(lambda: t.t.column(0)) / 1e9))
