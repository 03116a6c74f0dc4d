"""Host->device store upload bandwidth: raw pinned cudaMemcpy ceiling (torch)
vs DeviceStore.upload from pinned and pageable host memory (GPU box)."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_01409_b200 import _lib  # noqa: E402
from paper_1807_01409_b200.store import DeviceStore, TripleChunk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
ctx = _lib.context(0)
try:
    import torch

    a = torch.empty(n * 3, dtype=torch.int32, pin_memory=True)
    b = torch.empty(n * 3, dtype=torch.int32, device="cuda")
    for _ in range(2):
        b.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        b.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
    print(f"torch pinned H2D: {n * 12 * 5 / (time.perf_counter() - t) / 1e9:.1f} GB/s")
    del a, b
except Exception as e:  # noqa: BLE001
    print("torch probe failed:", e)
p = ctypes.c_void_p()
_lib.call("tidq_host_alloc", n * 12, ctypes.byref(p))
pinned = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint32)), shape=(n * 3,))
pinned[:] = np.arange(1, n * 3 + 1, dtype=np.uint32)
pageable = pinned.copy()
for name, arr in (("pinned", pinned), ("pageable", pageable)):
    ch = TripleChunk(arr, 0)
    DeviceStore.upload(ch).free()
    t = time.perf_counter()
    for _ in range(3):
        DeviceStore.upload(ch).free()
    dt = (time.perf_counter() - t) / 3
    print(f"DeviceStore.upload {name}: {n * 12 / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms for {n * 12 / 1e9:.2f} GB)")
ds = DeviceStore.upload(TripleChunk(pinned, 0))
got = ds.download(0, 1000)
assert np.array_equal(got.reshape(-1), pinned[:3000]), "upload mismatch"
got = ds.download(n - 1000, 1000)
assert np.array_equal(got.reshape(-1), pinned[-3000:]), "upload mismatch (tail)"
print("upload verified")

# native .tid ingest (file in the page cache after the write)
import tempfile  # noqa: E402

from paper_1807_01409_b200.store import write_tid  # noqa: E402

with tempfile.TemporaryDirectory() as td:
    path = os.path.join(td, "store.tid")
    write_tid(pinned.reshape(-1, 3), path)
    DeviceStore.load(path).free()
    t = time.perf_counter()
    for _ in range(3):
        DeviceStore.load(path).free()
    dt = (time.perf_counter() - t) / 3
    print(f"DeviceStore.load(.tid, page cache): {n * 12 / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)")
