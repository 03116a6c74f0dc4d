"""tidq — B200-native TripleID-Q query hot path (arXiv 1807.01409).

Drop-in for the reference ``tripleid`` package's load/query operator API
(``tripleid.kernel``, ``tripleid.query_ops``, ``tripleid.store``) backed by
hand-written sm_100a CUDA kernels in ``libtidq.so`` (C ABI: include/tidq.h).

    from paper_1807_01409_b200 import kernel, query_ops, store
    ds = store.DeviceStore.upload(chunk)               # resident SoA in HBM
    res = kernel.search_multi(ds, keys)                 # MatchResult
    table = query_ops.evaluate_query(compiled, ds, dictionary)
"""

from . import errors, plan, synth  # noqa: F401  (no native code needed)

__version__ = "0.1.0"


def __getattr__(name):
    # lazy: importing these loads nothing native until a call is made
    import importlib

    if name in ("kernel", "store", "query_ops", "distributed", "entailment", "_lib"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
