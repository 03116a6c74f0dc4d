"""CPU engine for the sharded planner (paper_1807_01409_b200.distributed):
oracle operators on numpy tables + torch.distributed ``gloo`` exchanges.

Test infrastructure only — it lets the world_size>1 planner logic (join
plans, partitioning, global row cap, DISTINCT exchange) run on CPU and be
compared against the reference's golden results.  The partition hash is the
product's ``partition_dest`` (the host statement of csrc/comm.cu)."""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from oracle import query as oq
from oracle import scan as oscan
from paper_1807_01409_b200.distributed import partition_dest
from paper_1807_01409_b200.errors import ResourceLimit


class GlooOracleEngine:
    def __init__(self, chunk, dictionary):
        self.chunk, self.dictionary = chunk, dictionary
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.exchanges = []  # ("shuffle" | "replicate", columns) log for plan checks

    # -- local operators (oracle) ---------------------------------------------------
    def scan(self, compiled):
        per_group = oscan.scan_patterns(compiled.groups, self.chunk)
        out = []
        for cg, rows in zip(compiled.groups, per_group):
            tables = [oq.pattern_table(p, vs, r) for p, vs, r in zip(cg.patterns, cg.var_slots, rows)]
            for flt in cg.filters:
                tables = [oq.apply_filter(t, flt.variable, flt.regex, self.dictionary)
                          if flt.variable in t.data else t for t in tables]
            out.append(tables)
        return out

    @staticmethod
    def n_rows(t):
        return t.n_rows

    @staticmethod
    def columns(t):
        return list(t.columns)

    def join(self, left, right, var, row_cap):
        """One step of oracle join_group (query_ops.py:318-341)."""
        pairs = oq.merge_join(left.data[var], right.data[var])
        if row_cap is not None and len(pairs) > row_cap:
            raise ResourceLimit(f"join produced {len(pairs)} rows, cap is {row_cap}")
        li, ri = pairs[:, 0], pairs[:, 1]
        cols = list(left.columns)
        data = {c: left.data[c][li] for c in left.columns}
        keep = None
        for c in right.columns:
            if c == var:
                continue
            rc = right.data[c][ri]
            if c in data:
                eq = data[c] == rc
                keep = eq if keep is None else keep & eq
            else:
                cols.append(c)
                data[c] = rc
        out = oq.Table(cols, data)
        if keep is not None:
            out = out.take(np.flatnonzero(keep))
        return out, len(pairs)

    def union(self, tables):
        return oq.evaluate_union(tables)

    def project(self, t, cols):
        return oq.project_distinct(t, cols, False) if cols else oq.Table([], {})

    def distinct(self, t, cols):
        return oq.project_distinct(t, cols, True)

    # -- exchanges (gloo) -----------------------------------------------------------
    def shuffle(self, t, key_cols):
        self.exchanges.append(("shuffle", tuple(key_cols)))
        if not t.columns:
            return t
        dest = partition_dest([t.data[c] for c in key_cols], self.world)
        order = np.argsort(dest, kind="stable")
        send = np.bincount(dest, minlength=self.world).astype(np.int64)
        recv = torch.zeros(self.world, dtype=torch.int64)
        dist.all_to_all_single(recv, torch.from_numpy(send))
        recv = recv.tolist()
        data = {}
        for c in t.columns:
            src = torch.from_numpy(t.data[c][order].astype(np.int64))
            dst = torch.empty(sum(recv), dtype=torch.int64)
            dist.all_to_all_single(dst, src, output_split_sizes=recv, input_split_sizes=send.tolist())
            data[c] = dst.numpy().astype(np.uint32)
        return oq.Table(list(t.columns), data)

    def replicate(self, t):
        self.exchanges.append(("replicate", tuple(t.columns)))
        return self._allgather(t)

    def _allgather(self, t):
        parts = [None] * self.world
        dist.all_gather_object(parts, (list(t.columns), {c: t.data[c] for c in t.columns}))
        cols = parts[0][0]
        return oq.Table(cols, {c: np.concatenate([p[1][c] for p in parts]).astype(np.uint32) for c in cols})

    def allreduce(self, values):
        x = torch.tensor([int(v) for v in values], dtype=torch.int64)
        dist.all_reduce(x)
        return [int(v) for v in x.tolist()]

    def collect(self, t):
        if not t.columns:
            return t
        return self._allgather(t)


class GlooStagedComm:
    """The DeviceEngine's communicator interface over gloo with host staging:
    the partition is the device kernel (tidq_table_partition), the exchanges
    download, move the rows over torch.distributed gloo and upload them.
    Test infrastructure only — it lets several ranks share ONE GPU (NCCL
    needs a device per rank), so the device engine's multi-rank planner path
    (row-sharded device scans, device partitions, device joins / DISTINCT)
    runs on the hardware at world_size > 1."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def partition(self, t, key_cols):
        from paper_1807_01409_b200.distributed import partition_table

        return partition_table(t, list(key_cols), self.world)

    def alltoallv(self, t, send_counts):
        from paper_1807_01409_b200.query_ops import DevTable

        send = np.asarray(send_counts, dtype=np.int64)
        recv = torch.zeros(self.world, dtype=torch.int64)
        dist.all_to_all_single(recv, torch.from_numpy(send))
        recv = recv.tolist()
        host = t.download()
        data = {}
        for c in t.columns:
            src = torch.from_numpy(host.data[c].astype(np.int64))
            dst = torch.empty(sum(recv), dtype=torch.int64)
            dist.all_to_all_single(dst, src, output_split_sizes=recv, input_split_sizes=send.tolist())
            data[c] = dst.numpy().astype(np.uint32)
        return DevTable.upload(list(t.columns), data, self.ctx)

    def allgather(self, t):
        from paper_1807_01409_b200.query_ops import DevTable

        host = t.download()
        parts = [None] * self.world
        dist.all_gather_object(parts, {c: host.data[c] for c in t.columns})
        return DevTable.upload(list(t.columns), {c: np.concatenate([p[c] for p in parts]).astype(np.uint32)
                                                 for c in t.columns}, self.ctx)

    def allreduce(self, values):
        x = torch.tensor([int(v) for v in values], dtype=torch.int64)
        dist.all_reduce(x)
        return [int(v) for v in x.tolist()]
