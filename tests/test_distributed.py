"""Multi-rank planner (paper_1807_01409_b200.distributed) on CPU: world_size
2 and 3 over gloo, row-sharded golden datasets, every golden query case under
forced BROADCAST and forced SHUFFLE join plans — multiset parity with the
reference's golden results, identical exceptions on every rank."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import IdDictionary, load_golden, plan_from_json, sorted_rows, table_rows
from paper_1807_01409_b200.distributed import partition_dest, shard_bounds
from paper_1807_01409_b200.store import TripleChunk
from paper_1807_01409_b200.synth import SynthDictionary


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dataset(meta, arrays, name, world, rank):
    d = meta[f"dataset_{name}"]
    rows = arrays[d["data"]].reshape(-1, 3)
    lo, hi = shard_bounds(len(rows), world, rank)
    chunk = TripleChunk(np.ascontiguousarray(rows[lo:hi]).reshape(-1), lo)
    dictionary = SynthDictionary(d["n_p"], d["n_e"]) if name == "a" else IdDictionary(d["max_id"])
    return chunk, dictionary


def _worker(rank, world, port, broadcast_rows_list):
    from dist_engine import GlooOracleEngine
    from paper_1807_01409_b200.distributed import evaluate_query_sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        meta, arrays = load_golden()
        failures = []
        plans_seen = set()
        for case in meta["query"]:
            chunk, dictionary = _dataset(meta, arrays, case["dataset"], world, rank)
            compiled = plan_from_json(case["plan"])
            for brows in broadcast_rows_list:
                eng = GlooOracleEngine(chunk, dictionary)
                try:
                    res = evaluate_query_sharded(compiled, eng, row_cap=case["row_cap"], broadcast_rows=brows)
                    res = eng.collect(res)
                    err = None
                except Exception as e:  # every rank must raise the same type
                    err = type(e).__name__
                plans_seen |= {kind for kind, _ in eng.exchanges}
                tag = f"{case['name']} world={world} broadcast_rows={brows}"
                if "error" in case:
                    if err != case["error"]:
                        failures.append(f"{tag}: expected {case['error']}, got {err}")
                    continue
                if err is not None:
                    failures.append(f"{tag}: raised {err}")
                    continue
                if list(res.columns) != case["columns"]:
                    failures.append(f"{tag}: columns {res.columns} != {case['columns']}")
                    continue
                want = arrays[case["result"]].reshape(case["n_rows"], -1)
                got = table_rows(res).reshape(-1, want.shape[1]) if res.columns else table_rows(res)
                if got.shape != want.shape or not np.array_equal(sorted_rows(got), sorted_rows(want)):
                    failures.append(f"{tag}: {got.shape[0]} rows, want {want.shape[0]} (multiset differs)")
        if world > 1 and {"shuffle", "replicate"} - plans_seen:
            failures.append(f"plans not exercised: {plans_seen}")
        if failures:
            raise AssertionError(f"rank {rank}: " + "; ".join(failures[:10]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_planner_matches_golden(world):
    # broadcast_rows 0 forces hash SHUFFLE joins; a large one forces BROADCAST
    mp.spawn(_worker, args=(world, _free_port(), [0, 1 << 30]), nprocs=world, join=True)


def test_partition_hash_statement():
    """dest = ((h >> 32) % world) with h = fold((h ^ v) * 0x9E3779B97F4A7C15)."""
    a = np.array([0, 1, 2, 0xFFFFFFFF, 12345], dtype=np.uint32)
    b = np.array([7, 7, 7, 7, 7], dtype=np.uint32)
    m = (1 << 64) - 1
    for world in (1, 2, 3, 8):
        want = []
        for x, y in zip(a.tolist(), b.tolist()):
            h = 0
            for v in (x, y):
                h = ((h ^ v) * 0x9E3779B97F4A7C15) & m
            want.append((h >> 32) % world)
        np.testing.assert_array_equal(partition_dest([a, b], world), want)


def test_shard_bounds_cover():
    for n in (0, 1, 7, 100):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
