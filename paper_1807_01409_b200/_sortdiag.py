"""Diagnostics for the device radix sort (tests and tools/sort_bench.py only):
sort host (key, value) pairs through tidq_debug_radix_sort and optionally
time device sorts.  Not part of the reference-facing API."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def radix_sort(keys: np.ndarray, vals: np.ndarray, bits: int, reps: int = 0):
    """Return (sorted keys, carried values, ms per device sort or 0.0)."""
    keys = np.ascontiguousarray(keys).copy()
    vals = np.ascontiguousarray(vals, dtype=np.uint32).copy()
    if keys.dtype not in (np.uint32, np.uint64):
        raise TypeError("keys must be uint32 or uint64")
    if len(keys) != len(vals):
        raise ValueError("keys and vals differ in length")
    ms = ctypes.c_double(0.0)
    _lib.call("tidq_debug_radix_sort", _lib.context().handle, keys.dtype.itemsize, _lib.ptr(keys), _lib.ptr(vals),
              len(keys), int(bits), int(reps), ctypes.byref(ms))
    return keys, vals, ms.value
