"""GPU: the multi-GPU exchange layer of libtidq (csrc/comm.cu) on one B200.

* tidq_table_partition against the host statement of the hash
  (distributed.partition_dest) for 1..8 ranks and 1..4 key columns — exact
  counts and stable grouping;
* a world_size-1 NCCL communicator: alltoallv / allgather / allreduce are
  identities;
* the sharded planner with the device engine (world 1) on every golden query
  case against the reference's golden results;
* the device engine at world_size 2 and 3 on the one GPU: every rank a
  process with its row shard resident, device scans / partitions / joins /
  DISTINCT, the exchanges staged through the host over gloo (NCCL needs a
  GPU per rank) — multiset parity with the golden results under forced
  SHUFFLE and BROADCAST join plans.
The world_size>1 planner logic also runs on CPU in tests/test_distributed.py."""

import numpy as np
import pytest

from helpers import IdDictionary, load_golden, plan_from_json, sorted_rows, table_rows
from paper_1807_01409_b200 import query_ops as Q
from paper_1807_01409_b200.distributed import (Communicator, DeviceEngine, evaluate_query_sharded, partition_dest,
                                               partition_table)
from paper_1807_01409_b200.store import DeviceStore, TripleChunk
from paper_1807_01409_b200.synth import SynthDictionary

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm(gpu):
    c = Communicator(gpu, 0, 1, Communicator.unique_id())
    yield c
    c.close()


@pytest.mark.parametrize("nkeys", [1, 2, 3, 4])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_matches_host_hash(gpu, world, nkeys):
    rng = np.random.default_rng(world * 10 + nkeys)
    n = 300_000
    cols = [f"c{i}" for i in range(5)]
    data = {c: rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32) for c in cols}
    data["c0"][:1000] = 0  # UNBOUND values hash too
    t = Q.DevTable.upload(cols, data, gpu)
    parted, counts = partition_table(t, cols[:nkeys], world)
    dest = partition_dest([data[c] for c in cols[:nkeys]], world)
    np.testing.assert_array_equal(counts, np.bincount(dest, minlength=world))
    order = np.argsort(dest, kind="stable")
    got = parted.download()
    for c in cols:
        np.testing.assert_array_equal(got.data[c], data[c][order])


def test_comm_world1_identities(gpu, comm):
    rng = np.random.default_rng(1)
    data = {"a": rng.integers(0, 2**32, size=123_457, dtype=np.uint64).astype(np.uint32),
            "b": rng.integers(0, 50, size=123_457).astype(np.uint32)}
    t = Q.DevTable.upload(["a", "b"], data, gpu)
    for out in (comm.alltoallv(t, np.array([t.n_rows], np.uint64)), comm.allgather(t)):
        got = out.download()
        for c in ("a", "b"):
            np.testing.assert_array_equal(got.data[c], data[c])
    assert comm.allreduce([3, 2**40, 0]) == [3, 2**40, 0]
    empty = Q.DevTable.upload(["a"], {"a": np.empty(0, np.uint32)}, gpu)
    assert comm.alltoallv(empty, np.zeros(1, np.uint64)).n_rows == 0
    assert comm.allgather(empty).n_rows == 0


def test_sharded_planner_device_golden(gpu, comm):
    meta, arrays = load_golden()
    stores = {}
    for name in ("a", "b", "c", "d"):
        d = meta[f"dataset_{name}"]
        rows = arrays[d["data"]].reshape(-1)
        dictionary = SynthDictionary(d["n_p"], d["n_e"]) if name == "a" else IdDictionary(d["max_id"])
        stores[name] = (DeviceStore.upload(TripleChunk(rows, 0)), dictionary)
    for case in meta["query"]:
        ds, dictionary = stores[case["dataset"]]
        eng = DeviceEngine(ds, dictionary, comm)
        compiled = plan_from_json(case["plan"])
        if "error" in case:
            with pytest.raises(Exception) as ei:
                evaluate_query_sharded(compiled, eng, row_cap=case["row_cap"])
            assert type(ei.value).__name__ == case["error"], case["name"]
            continue
        res = eng.collect(evaluate_query_sharded(compiled, eng, row_cap=case["row_cap"]))
        assert list(res.columns) == case["columns"], case["name"]
        want = arrays[case["result"]].reshape(case["n_rows"], -1)
        got = table_rows(res).reshape(-1, want.shape[1])
        np.testing.assert_array_equal(sorted_rows(got), sorted_rows(want), err_msg=case["name"])


def test_comm_stats_world1(gpu, comm):
    """exchange accounting: nothing leaves the GPU at world size 1"""
    rng = np.random.default_rng(4)
    t = Q.DevTable.upload(["a"], {"a": rng.integers(1, 1000, size=5000, dtype=np.uint64).astype(np.uint32)}, gpu)
    comm.stats(reset=True)
    parted, counts = comm.partition(t, ["a"])
    out = comm.alltoallv(parted, counts)
    assert out.n_rows == 5000
    sent, ms = comm.stats(reset=True)
    assert sent == 0 and ms >= 0


def test_engine_from_tid_shard(gpu, comm, golden, tmp_path):
    """DeviceEngine.from_tid: the rank's row shard of a .tid file (world 1:
    the whole file) through the sharded planner equals the golden result."""
    from paper_1807_01409_b200.store import write_tid

    meta, arrays = golden
    d = meta["dataset_a"]
    p = tmp_path / "a.tid"
    write_tid(arrays[d["data"]], p)
    dictionary = SynthDictionary(d["n_p"], d["n_e"])
    engine = DeviceEngine.from_tid(p, dictionary, comm)
    assert len(engine.store) == d["n"] and engine.store.base_index == 0
    n = 0
    for case in meta["query"]:
        if case["dataset"] != "a" or "error" in case:
            continue
        t = engine.collect(evaluate_query_sharded(plan_from_json(case["plan"]), engine, row_cap=case["row_cap"]))
        want = arrays[case["result"]]
        np.testing.assert_array_equal(sorted_rows(table_rows(t).reshape(want.shape)), sorted_rows(want),
                                      err_msg=case["name"])
        n += 1
    assert n >= 10
    engine.store.free()


def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _device_worker(rank, world, port):
    import torch.distributed as dist

    from dist_engine import GlooStagedComm
    from paper_1807_01409_b200 import _lib
    from paper_1807_01409_b200.distributed import shard_bounds

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        ctx = _lib.context(0)
        comm = GlooStagedComm(ctx)
        meta, arrays = load_golden()
        stores = {}
        for name in ("a", "b", "c", "d"):
            d = meta[f"dataset_{name}"]
            rows = arrays[d["data"]].reshape(-1, 3)
            lo, hi = shard_bounds(len(rows), world, rank)
            dictionary = SynthDictionary(d["n_p"], d["n_e"]) if name == "a" else IdDictionary(d["max_id"])
            stores[name] = (DeviceStore.upload(TripleChunk(np.ascontiguousarray(rows[lo:hi]).reshape(-1), lo)),
                            dictionary)
        failures = []
        for case in meta["query"]:
            ds, dictionary = stores[case["dataset"]]
            compiled = plan_from_json(case["plan"])
            for brows in (0, 1 << 30):  # forced SHUFFLE / forced BROADCAST joins
                eng = DeviceEngine(ds, dictionary, comm)
                tag = f"{case['name']} world={world} broadcast_rows={brows}"
                try:
                    res = eng.collect(evaluate_query_sharded(compiled, eng, row_cap=case["row_cap"],
                                                             broadcast_rows=brows))
                    err = None
                except Exception as e:  # every rank must raise the same type
                    err = type(e).__name__
                if "error" in case:
                    if err != case["error"]:
                        failures.append(f"{tag}: expected {case['error']}, got {err}")
                    continue
                if err is not None:
                    failures.append(f"{tag}: raised {err}")
                    continue
                if list(res.columns) != case["columns"]:
                    failures.append(f"{tag}: columns {res.columns}")
                    continue
                want = arrays[case["result"]].reshape(case["n_rows"], -1)
                got = table_rows(res).reshape(-1, want.shape[1]) if res.columns else table_rows(res)
                if got.shape != want.shape or not np.array_equal(sorted_rows(got), sorted_rows(want)):
                    failures.append(f"{tag}: {got.shape[0]} rows, want {want.shape[0]}")
        if failures:
            raise AssertionError(f"rank {rank}: " + "; ".join(failures[:10]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_device_engine_multi_rank(gpu, world):
    import torch.multiprocessing as mp

    mp.spawn(_device_worker, args=(world, _free_port()), nprocs=world, join=True)
