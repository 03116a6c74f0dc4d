"""Row-sharded, multi-GPU evaluation of the TripleID-Q query path.

The reference evaluates a query in one process: a chunked scan of the whole
store (query_ops.py:263-295), a left-deep chain of merge joins per UNION
branch (query_ops.py:298-342), UNION concatenation (query_ops.py:359-376) and
projection/DISTINCT (query_ops.py:379-399).  Here the store is split into
contiguous row shards, one per rank (one process per GPU), and:

* the scan is local — every rank scans only its shard, no communication;
* each join step is local once both inputs are co-partitioned on the join
  variable.  The planner picks, identically on every rank from an allreduce
  of the two global sizes,
    - BROADCAST: the smaller side (global rows <= ``broadcast_rows``) is
      all-gathered to every rank and joined with the other side's local
      shard.  Each output pair is produced exactly once (the large side is
      partitioned), and the large side keeps its partitioning;
    - SHUFFLE: both sides are hash-partitioned on the join variable and
      exchanged with a variable-size all-to-all, then joined locally.  The
      result stays partitioned on that variable, so a later step on the same
      variable (star queries) shuffles only the new pattern table;
* the row cap (query_ops.py:330-334) is checked on the GLOBAL pair count
  (allreduce of the local counts) so every rank raises ResourceLimit
  together;
* UNION is a local concatenation;
* DISTINCT is local when every branch is already partitioned on a projected
  variable; otherwise rows are deduplicated locally, hash-partitioned on the
  projected columns, exchanged, and deduplicated again.

Results are a MULTISET match of the single-process reference (row order is
by owner rank); DISTINCT results are the same set.  The hash used for every
partitioning is the one libtidq implements (csrc/comm.cu):

    h = 0;  for v in key columns: h = (h ^ v) * 0x9E3779B97F4A7C15 (mod 2^64)
    dest = (h >> 32) % world

The planner is written against a small engine interface.  ``DeviceEngine``
is the product: libtidq device tables on the local GPU and a libtidq-owned
NCCL communicator (``Communicator``) for the exchanges.  The tests drive the
same planner with a CPU engine over ``gloo`` (tests/dist_engine.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import query_ops as Q
from .errors import ResourceLimit
from .query_ops import DEFAULT_ROW_CAP, BindingTable, DevTable, analyze_relationships
from .store import DeviceStore

__all__ = [
    "HASH_MULT",
    "partition_dest",
    "partition_table",
    "shard_bounds",
    "Communicator",
    "DeviceEngine",
    "evaluate_query_sharded",
]

HASH_MULT = 0x9E3779B97F4A7C15
MAX_PARTITION_KEYS = 4
DEFAULT_BROADCAST_ROWS = 1 << 20


def partition_dest(key_columns, world: int) -> np.ndarray:
    """Host statement of the device partition hash (csrc/comm.cu dest_kernel)."""
    cols = [np.asarray(c, dtype=np.uint64) for c in key_columns[:MAX_PARTITION_KEYS]]
    n = len(cols[0]) if cols else 0
    h = np.zeros(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for c in cols:
            h = (h ^ c) * np.uint64(HASH_MULT)
    return ((h >> np.uint64(32)) % np.uint64(world)).astype(np.int64)


def shard_bounds(n_triples: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row shard [lo, hi) of ``rank`` (sizes differ by at most 1)."""
    q, r = divmod(int(n_triples), world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


# ----------------------------------------------------------------------------- planner

@dataclass
class _Part:
    """A local table and how its rows are spread over the ranks: ``key`` is
    None (arbitrary, e.g. scan shards) or the variable it is hash-partitioned
    on."""

    table: object
    key: str | None = None


def _join_step(engine, acc: _Part, right: _Part, var: str, row_cap, broadcast_rows: int) -> _Part:
    n_acc, n_right = engine.allreduce([engine.n_rows(acc.table), engine.n_rows(right.table)])
    if engine.world == 1:
        plan = "local"
    elif acc.key == var and right.key == var:
        plan = "local"
    elif min(n_acc, n_right) <= broadcast_rows:
        plan = "bcast_right" if n_right <= n_acc else "bcast_left"
    else:
        plan = "shuffle"
    left_t, right_t, out_key = acc.table, right.table, acc.key
    if plan == "bcast_right":
        right_t = engine.replicate(right_t)
    elif plan == "bcast_left":
        left_t, out_key = engine.replicate(left_t), right.key
    elif plan == "shuffle":
        if acc.key != var:
            left_t = engine.shuffle(left_t, [var])
        if right.key != var:
            right_t = engine.shuffle(right_t, [var])
        out_key = var
    elif engine.world > 1:
        out_key = var
    try:
        out, pairs = engine.join(left_t, right_t, var, row_cap)
    except ResourceLimit:
        out, pairs = None, (row_cap or 0) + 1
    (total,) = engine.allreduce([pairs])
    if row_cap is not None and total > row_cap:
        raise ResourceLimit(f"join produced {total} rows across {engine.world} ranks, cap is {row_cap}")
    return _Part(out, out_key)


def evaluate_query_sharded(compiled, engine, row_cap: int | None = DEFAULT_ROW_CAP,
                           broadcast_rows: int = DEFAULT_BROADCAST_ROWS):
    """evaluate_query (query_ops.py:432-455) over row shards.  Returns this
    rank's share of the result as an engine table with the query's output
    columns; ``engine.collect`` gathers the whole result."""
    per_group = engine.scan(compiled)
    branches = []
    for cg, tables in zip(compiled.groups, per_group):
        rels = analyze_relationships(cg.patterns)
        acc = _Part(tables[0])
        for rel in rels:
            acc = _join_step(engine, acc, _Part(tables[rel.j]), rel.variable, row_cap, broadcast_rows)
        branches.append(acc)
    union = engine.union([b.table for b in branches])
    union_cols = engine.columns(union)
    cols = list(compiled.projection) if compiled.projection is not None else list(union_cols)
    missing = [c for c in cols if c not in union_cols]
    if missing:
        raise KeyError(f"projection names unbound variables: {missing}")
    out = engine.project(union, cols)
    if not compiled.distinct or not cols:
        return out
    keys = {b.key for b in branches}
    if engine.world > 1 and not (len(keys) == 1 and next(iter(keys)) in cols):
        out = engine.distinct(out, cols)
        out = engine.shuffle(out, cols)
    return engine.distinct(out, cols)


# ----------------------------------------------------------------------------- device engine


def partition_table(t: DevTable, key_cols: list, world: int) -> tuple[DevTable, np.ndarray]:
    """Rows of ``t`` grouped by destination rank (stable within a rank) and
    the per-rank row counts (tidq_table_partition)."""
    idx = [t.col(c) for c in key_cols[:MAX_PARTITION_KEYS]]
    counts = np.zeros(world, dtype=np.uint64)
    h = ctypes.c_void_p()
    _lib.call("tidq_table_partition", t.t.handle, len(idx), Q._i32(idx), int(world), ctypes.byref(h),
              _lib.ptr(counts))
    return DevTable.from_handle(t.columns, h), counts


class Communicator:
    """A libtidq NCCL communicator over the ranks of one job (tidq_comm)."""

    ID_BYTES = 128

    def __init__(self, ctx: _lib.Context, rank: int, world: int, unique_id: bytes):
        if len(unique_id) != self.ID_BYTES:
            raise ValueError("unique id must be 128 bytes")
        self.ctx, self.rank, self.world = ctx, int(rank), int(world)
        buf = (ctypes.c_uint8 * self.ID_BYTES).from_buffer_copy(unique_id)
        h = ctypes.c_void_p()
        _lib.call("tidq_comm_create", ctx.handle, buf, self.world, self.rank, ctypes.byref(h))
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * Communicator.ID_BYTES)()
        _lib.call("tidq_comm_unique_id", buf)
        return bytes(buf)

    @classmethod
    def from_torch(cls, ctx: _lib.Context | None = None) -> "Communicator":
        """Bootstrap over an initialised torch.distributed process group
        (rank 0 creates the id, a broadcast hands it to the others)."""
        import torch.distributed as dist

        ctx = ctx or _lib.context()
        rank, world = dist.get_rank(), dist.get_world_size()
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        return cls(ctx, rank, world, box[0])

    def stats(self, reset: bool = False) -> tuple[int, float]:
        """(payload bytes sent to other ranks, device ms of the exchanges)."""
        b, ms = ctypes.c_uint64(), ctypes.c_double()
        _lib.call("tidq_comm_stats", self.handle, int(reset), ctypes.byref(b), ctypes.byref(ms))
        return b.value, ms.value

    def close(self) -> None:
        if self.handle is not None and self.handle.value:
            _lib.call("tidq_comm_destroy", self.handle)
        self.handle = None

    # -- table exchanges --------------------------------------------------------
    def partition(self, t: DevTable, key_cols: list) -> tuple[DevTable, np.ndarray]:
        return partition_table(t, key_cols, self.world)

    def alltoallv(self, t: DevTable, send_counts: np.ndarray) -> DevTable:
        send = np.ascontiguousarray(send_counts, dtype=np.uint64)
        recv = np.zeros(self.world, dtype=np.uint64)
        h = ctypes.c_void_p()
        _lib.call("tidq_table_alltoallv", self.handle, t.t.handle, _lib.ptr(send), ctypes.byref(h),
                  _lib.ptr(recv))
        return DevTable.from_handle(t.columns, h)

    def allgather(self, t: DevTable) -> DevTable:
        return DevTable.from_handle(t.columns, Q._new_handle("tidq_table_allgather", self.handle, t.t.handle))

    def allreduce(self, values) -> list:
        a = np.ascontiguousarray(values, dtype=np.uint64)
        out = np.zeros_like(a)
        _lib.call("tidq_comm_allreduce_u64", self.handle, _lib.ptr(a), _lib.ptr(out), len(a))
        return [int(x) for x in out]


class DeviceEngine:
    """Planner engine over libtidq: the local shard is a resident DeviceStore,
    tables are DevTables on this rank's GPU, exchanges go over NCCL."""

    def __init__(self, store: DeviceStore, dictionary, comm: Communicator):
        self.store, self.dictionary, self.comm = store, dictionary, comm
        self.rank, self.world = comm.rank, comm.world

    @classmethod
    def from_tid(cls, path, dictionary, comm: Communicator) -> "DeviceEngine":
        """Each rank loads its contiguous row shard of a ``.tid`` file
        (tidq_store_load_tid_range) onto its own GPU."""
        return cls(DeviceStore.load_shard(path, comm.rank, comm.world, device=comm.ctx.device),
                   dictionary, comm)

    def scan(self, compiled):
        # no semi-join reduction here: a row's partners may live on other ranks
        return Q._scan_device([(self.store, False)], compiled.groups, self.dictionary, fuse_filters=True,
                              compiled=compiled, reduce=False)

    @staticmethod
    def n_rows(t: DevTable) -> int:
        return t.n_rows

    @staticmethod
    def columns(t: DevTable) -> list:
        return list(t.columns)

    def join(self, left: DevTable, right: DevTable, var: str, row_cap):
        return Q._dev_join_counted(left, right, var, row_cap)

    def union(self, tables):
        return Q._union_device(list(tables)) if tables else DevTable([], None)

    def project(self, t: DevTable, cols):
        return Q._dev_project(t, list(cols)) if cols else DevTable([], None)

    def distinct(self, t: DevTable, cols):
        return Q._dev_distinct(t, list(cols)) if t.n_rows else Q._dev_project(t, list(cols))

    def shuffle(self, t: DevTable, key_cols):
        if not t.columns:
            return t
        parted, counts = self.comm.partition(t, list(key_cols))
        return self.comm.alltoallv(parted, counts)

    def replicate(self, t: DevTable):
        return self.comm.allgather(t) if t.columns else t

    def allreduce(self, values):
        return self.comm.allreduce(values)

    def collect(self, t: DevTable) -> BindingTable:
        """Every rank's rows, in rank order, on every rank."""
        if not t.columns:
            return BindingTable([], {})
        return self.comm.allgather(t).download()

