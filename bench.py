"""Benchmark: triple-pattern scan throughput on a resident 100M-triple store.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tidq|reference]

Workload (BASELINE.json configs[1], "C2"): a 100M-triple synthetic TripleID
store (Zipfian predicates: seed 2, n_p = 10^4, n_e = 10^7)
generated on the device; one STEP = the selectivity sweep of single-pattern
queries ``SELECT * WHERE { ?s <p/r> ?o }`` for predicate ranks
r in {1, 10, 100, 1000, 10000} (10.2 % ... 0.001 % selectivity), each through
``query_ops.evaluate_query`` on the resident store (scan + binding columns).
metric = triples scanned per second (5 x 10^8 triples per step per GPU).

Multi-GPU (torchrun): every rank holds its own 100M-triple row shard of a
N x 100M store (global indices rank*N...), scans it locally, no collective
on the data path -> weak scaling; times are max over ranks.

Timing: CUDA events on the libtidq stream, W warm-up steps, K timed steps
bracketed by barrier + device synchronisation; the 400 MB predicate column
is larger than the 126 MB L2, so every scan streams from HBM.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RANKS = [1, 10, 100, 1000, 10000]
N_TRIPLES = 100_000_000
N_P = 10_000
SEED = 2
OUT = sys.stdout  # the JSON line's stream (main() points it at the real stdout)
METRIC = "triples scanned/sec (single-pattern scan sweep, C2 100M Zipf store)"
UNIT = "triples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tidq", choices=["tidq", "reference"])
    ap.add_argument("--n-triples", type=int, default=N_TRIPLES)
    ap.add_argument("--cpu-sample", type=int, default=20_000_000,
                    help="triples in the bounded CPU-baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-join", action="store_true")
    ap.add_argument("--join-triples", type=int, default=2_000_000_000,
                    help="C5 store size (row-sharded over the ranks)")
    ap.add_argument("--join-reps", type=int, default=5)
    ap.add_argument("--join-timeout", type=float, default=240.0)
    ap.add_argument("--join-sharded", action="store_true",
                    help="use the NCCL sharded planner even at N=1 (exercises the multi-GPU path)")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the C3/C4/C5 per-query section (device, e2e, CPU baselines)")
    ap.add_argument("--configs", default="C3,C4,C5")
    ap.add_argument("--config-reps", type=int, default=5)
    ap.add_argument("--config-cpu-scale", type=float, default=0.01,
                    help="CPU baselines of C3-C5 run on the config scaled by this factor (N and n_e)")
    ap.add_argument("--configs-worker", default="",
                    help=argparse.SUPPRESS)  # internal: one config's section in a fresh process
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    ~2 ms during the timed region (nvidia-smi as a fallback)."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
               ("hw_power_brake_slowdown", 0x80), ("sw_power_cap", 0x4))

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, reasons_mask)
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                              "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip().split(",")
        self.max_mhz = float(out[1])
        return float(out[0]), int(out[2].strip(), 16)

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    nv = self._nvml
                    self.samples.append((float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)),
                                         int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))))
                else:
                    self.samples.append(self._sample_smi())
            except Exception:
                pass
            self._stop.wait(0.002 if self._nvml is not None else 0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no clock samples"]}
        sm = sorted(x[0] for x in self.samples)
        reasons = sorted({name for _, m in self.samples for name, bit in self.REASONS if m & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic():
    """DRAM bytes (read + write) per launch from the committed ncu --set full
    capture of one bench step (tools/ncu_summary.py -> profiles/)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_scan_summary.json")))
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


def queries(dictionary):
    from paper_1807_01409_b200 import plan

    return [plan.compile_query([plan.Group([plan.pattern("?s", f"<http://example.org/p/{r}>", "?o")], [])],
                               dictionary) for r in RANKS]


P_IRI = "<http://example.org/p/{}>"


def q_union(d, ranks, projection=None, distinct=False):
    """C3: UNION of single-pattern branches ?s P_r ?o (same variable names)."""
    from paper_1807_01409_b200 import plan

    groups = [plan.Group([plan.pattern("?s", P_IRI.format(r), "?o")], []) for r in ranks]
    return plan.compile_query(groups, d, distinct=distinct, projection=projection)


def q_star(d, ranks, flt=None):
    """C4/C5 star: ?s P_a ?o1 . ?s P_b ?o2 ... [FILTER regex(str(?o1), flt)]."""
    from paper_1807_01409_b200 import plan

    pats = [plan.pattern("?s", P_IRI.format(r), f"?o{i + 1}") for i, r in enumerate(ranks)]
    return plan.compile_query([plan.Group(pats, [plan.Filter("o1", flt)] if flt else [])], d)


def q_chain(d, ranks, flt=None):
    """C4/C5 chain: ?x P_a ?y . ?y P_b ?z ... [FILTER regex(str(?y), flt)]."""
    from paper_1807_01409_b200 import plan

    names = ["x", "y", "z", "w", "v"]
    pats = [plan.pattern(f"?{names[i]}", P_IRI.format(r), f"?{names[i + 1]}") for i, r in enumerate(ranks)]
    return plan.compile_query([plan.Group(pats, [plan.Filter("y", flt)] if flt else [])], d)


def config_queries(cfg):
    """(name, builder(dictionary) -> CompiledQuery, cold-FILTER e2e?) per
    BASELINE config: C3 UNION x4/x8 bag and DISTINCT (?s, ?s ?o) over ranks
    2..9; C4 star/chain x2..x4 at ranks {3,5,7,11} with and without
    FILTER(regex(str(?v), "7$")); C5 3-way star and chain at ranks {5,7,11}."""
    out = []
    if cfg == "C3":
        for k in (4, 8):
            rk = list(range(2, 2 + k))
            out.append((f"C3 UNION x{k} (bag)", lambda d, rk=rk: q_union(d, rk), False))
            out.append((f"C3 DISTINCT ?s UNION x{k}", lambda d, rk=rk: q_union(d, rk, ["s"], True), False))
            out.append((f"C3 DISTINCT ?s ?o UNION x{k}", lambda d, rk=rk: q_union(d, rk, ["s", "o"], True), False))
    elif cfg == "C4":
        for k in (2, 3, 4):
            rk = [3, 5, 7, 11][:k]
            out.append((f"C4 star x{k}", lambda d, rk=rk: q_star(d, rk), False))
            out.append((f"C4 star x{k} FILTER", lambda d, rk=rk: q_star(d, rk, "7$"), k == 2))
            out.append((f"C4 chain x{k}", lambda d, rk=rk: q_chain(d, rk), False))
            out.append((f"C4 chain x{k} FILTER", lambda d, rk=rk: q_chain(d, rk, "7$"), k == 2))
    elif cfg == "C5":
        out.append(("C5 star x3", lambda d: q_star(d, [5, 7, 11]), False))
        out.append(("C5 chain x3", lambda d: q_chain(d, [5, 7, 11]), False))
    return out


def dram_floor(ds, n, step_ms, peak):
    """The step's minimum DRAM traffic with this store layout, next to the
    algorithmic bytes: every query streams the 400 MB predicate column, and
    the emit's gathers of s and o cannot fetch less than the 128-B lines that
    hold a hit — at 10 % selectivity that is 97 % of both columns, however
    few bytes the rows need — plus the rows written.  The composite's
    algorithmic fraction is capped by algorithmic / floor; the step's time
    against floor / peak says how close the kernels run to the layout's limit."""
    hist = ds.predicate_counts()
    pb = 2.0 if ds.pcodes and os.environ.get("TIDQ_P16", "1") != "0" else 4.0  # predicate-code column
    so = ds.so and os.environ.get("TIDQ_SO", "1") != "0"  # (s, o) pairs: 16 per 128-B line
    floor = algo = 0.0
    for r in RANKS:
        h = float(hist[r])
        if so:
            gather = 128.0 * (n / 16.0) * (1.0 - (1.0 - h / n) ** 16)
        else:
            gather = 2 * 128.0 * (n / 32.0) * (1.0 - (1.0 - h / n) ** 32)  # 32 uint32 per 128-B line
        floor += pb * n + gather + 8.0 * h
        algo += pb * n + 16.0 * h
    t_floor_ms = floor / (peak * 1e9) * 1e3
    return {"bytes_per_step": floor, "algo_bytes_per_step": algo, "algo_over_floor": algo / floor,
            "floor_ms_at_peak": t_floor_ms, "step_frac_of_floor": t_floor_ms / step_ms if step_ms else None,
            "model": f"5 x ({pb:.0f} B x N predicate column + 128 B x "
                     + ("(s, o) pair lines holding a hit" if so else "s and o lines holding a hit")
                     + " + 8 B x rows)"}


def configs_section(args, ctx, peak):
    """BASELINE configs[2..4] (C3, C4, C5) on one GPU, per query:
    - device: ms per query (median / best of --config-reps, CUDA events on the
      library stream; result resident on the device), the row count, and the
      per-operator roofline from the library's own per-launch events
      (scan: 4 B x N x bound columns + emitted fields; join: 4 B x (left +
      right + output cells); distinct: w x M + w x U);
    - e2e: query_ops.evaluate_query (compiled query -> host BindingTable,
      D2H included) with the FILTER regex cache warm, and for the x2 FILTER
      queries once more with a COLD cache (a fresh dictionary object: the
      host regex over the dictionary's IDs is inside the timed region);
    - cpu: the reference's CPU path (oracle port with the reference's own
      per-key merge_join loop and per-row DISTINCT set, all host cores) on the
      same generator scaled by --config-cpu-scale (N and n_e both scaled, so
      selectivities and per-key fan-outs are the config's), with a linear
      extrapolation to the full size stated as such."""
    import numpy as np

    from oracle import query as oq
    from oracle import synth as osynth
    from paper_1807_01409_b200 import query_ops
    from paper_1807_01409_b200.store import DeviceStore, TripleChunk
    from paper_1807_01409_b200.synth import CONFIGS, SynthDictionary, zipf_cdf_table

    cores = len(os.sched_getaffinity(0))
    out = {"row_cap": "reference default (10^7)", "cpu_cores": cores, "cpu_scale": args.config_cpu_scale}
    for cfg in [c for c in args.configs.split(",") if c]:
        c = CONFIGS[cfg]
        t0 = time.perf_counter()
        ds = DeviceStore.generate(c["n_triples"], seed=c["seed"], n_p=c["n_p"], n_e=c["n_e"])
        d = SynthDictionary(c["n_p"], c["n_e"])
        gen_s = time.perf_counter() - t0
        ds.prepare()  # index columns built at load time, outside every timed region
        n_cpu = int(c["n_triples"] * args.config_cpu_scale)
        ne_cpu = max(1, int(c["n_e"] * args.config_cpu_scale))
        chunk = d_cpu = None
        if not args.no_cpu and n_cpu > 0:
            rows = osynth.generate(n_cpu, seed=c["seed"], n_p=c["n_p"], n_e=ne_cpu, cdf=zipf_cdf_table(c["n_p"]),
                                   threads=cores)
            chunk = TripleChunk(rows.reshape(-1), 0)
            d_cpu = SynthDictionary(c["n_p"], ne_cpu)
        recs = {}
        for name, build, cold in config_queries(cfg):
            q = build(d)
            t = query_ops.evaluate_query_device(q, ds, d)  # warm: pools, FILTER cache
            n_rows = t.n_rows
            t.t and t.t.free()
            ctx.profile_reset()
            ctx.profile(True)
            times = []
            for _ in range(args.config_reps):
                ctx.sync()
                ctx.timer_begin()
                t = query_ops.evaluate_query_device(q, ds, d)
                times.append(ctx.timer_end())
                t.t and t.t.free()
            ctx.profile(False)
            times.sort()
            rec = {"rows": n_rows, "device_ms": times[len(times) // 2], "device_ms_best": times[0]}
            ops = {}
            for op in ("scan", "join", "distinct"):
                ms, launches, nbytes = ctx.profile_read(op)
                if launches:
                    gbs = nbytes / (ms / 1e3) / 1e9
                    ops[op] = {"ms_per_query": ms / args.config_reps, "calls_per_query": launches / args.config_reps,
                               "algo_bytes_per_query": nbytes / args.config_reps, "achieved_gbs": gbs,
                               "frac": gbs / peak}
            rec["operators"] = ops
            # e2e, warm cache: the drop-in call with a host BindingTable result
            # (median of 3; the first call also grows the pinned result pool)
            e2e = []
            for _ in range(3):
                ctx.sync()
                t0 = time.perf_counter()
                bt = query_ops.evaluate_query(q, ds, d)
                e2e.append(1e3 * (time.perf_counter() - t0))
                rec["d2h_bytes"] = int(sum(bt.data[col].nbytes for col in bt.columns))
                del bt
            rec["e2e_ms"] = sorted(e2e)[1]
            if cold:
                d_cold = SynthDictionary(c["n_p"], c["n_e"])  # no regex cache for this object
                ctx.sync()
                t0 = time.perf_counter()
                bt = query_ops.evaluate_query(build(d_cold), ds, d_cold)
                rec["e2e_cold_filter_ms"] = 1e3 * (time.perf_counter() - t0)
                del bt
            if chunk is not None:
                qc = build(d_cpu)
                t0 = time.perf_counter()
                r = oq.evaluate_query(qc, chunk, d_cpu, workers=cores, faithful=True)
                cpu_s = time.perf_counter() - t0
                rec["cpu"] = {"ms": 1e3 * cpu_s, "rows": r.n_rows, "triples": n_cpu, "n_e": ne_cpu,
                              "ms_extrapolated_linear": 1e3 * cpu_s / args.config_cpu_scale,
                              "kind": "port (faithful merge_join loop + DISTINCT set)"}
            recs[name] = rec
        ds.free()
        out[cfg] = {"store_triples": c["n_triples"], "n_e": c["n_e"], "seed": c["seed"],
                    "generate_s": round(gen_s, 2), "queries": recs}
    return out


def configs_in_workers(args):
    """configs_section, each config in a fresh process: a config's device
    times then do not depend on the pooled memory and host state the previous
    sections left behind (measured: C3 DISTINCT ?s UNION x4 3.8-10 ms after the
    C2 section in one process vs 2.9-3.0 ms in a fresh one)."""
    out = None
    for cfg in [c for c in args.configs.split(",") if c]:
        cmd = [sys.executable, os.path.abspath(__file__), "--configs-worker", cfg,
               "--config-reps", str(args.config_reps), "--config-cpu-scale", str(args.config_cpu_scale)]
        if args.no_cpu:
            cmd.append("--no-cpu")
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, env=os.environ.copy())
            sec = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as e:  # noqa: BLE001 - reported in the line, the scan metric stands
            sec = {cfg: {"error": f"{type(e).__name__}: {e}"[:300]}}
        if out is None:
            out = {k: v for k, v in sec.items() if k not in ("C3", "C4", "C5")}
            out["isolation"] = "each config in a fresh process (bench.py --configs-worker)"
        out[cfg] = sec.get(cfg, sec)
    return out


def run_configs_worker(args):
    from paper_1807_01409_b200 import _lib

    args.configs = args.configs_worker
    ctx = _lib.context(0)
    peak = measured_peaks().get("hbm_gbs") or 6650.0
    try:
        sec = configs_section(args, ctx, peak)
    except Exception as e:  # noqa: BLE001
        sec = {args.configs_worker: {"error": f"{type(e).__name__}: {e}"[:300]}}
    print(json.dumps(sec), file=OUT, flush=True)


def cpu_baseline(n_sample: int, dictionary, qs, min_seconds: float = 10.0):
    """The reference's CPU algorithm (oracle port) on a bounded sample of the
    same workload, all host cores as workers."""
    import numpy as np

    from oracle import query as oq
    from oracle import synth as osynth
    from paper_1807_01409_b200.store import TripleChunk
    from paper_1807_01409_b200.synth import zipf_cdf_table

    cores = len(os.sched_getaffinity(0))
    rows = osynth.generate(n_sample, seed=SEED, n_p=N_P, n_e=N_TRIPLES // 10, cdf=zipf_cdf_table(N_P))
    chunk = TripleChunk(rows.reshape(-1), 0)
    runs = 0
    t0 = time.perf_counter()
    while True:
        for q in qs:
            oq.evaluate_query(q, chunk, dictionary, workers=cores, row_cap=None)
        runs += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or runs >= 20:
            break
    value = runs * len(qs) * n_sample / el
    return {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"first {n_sample:,} triples of the C2 generator (seed {SEED}), the 5-query rank sweep "
                      f"x{runs} through oracle.query.evaluate_query (numpy restatement of the reference's "
                      f"search_multi tile pool + query_ops), workers={cores}",
            "seconds": round(el, 3)}, np


def run_reference(args):
    """The reference's CPU path (the oracle port: numpy restatement of
    search_multi's tile pool + query_ops) on the SAME workload as the GPU arm:
    the full C2 store (default 100M triples), every host core as a worker.
    One step = one query of the rank sweep over the whole store (cycling
    through the 5 ranks), so K + W steps finish within a few minutes; the
    metric (triples scanned per second) is a rate either way."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import query as oq
    from oracle import synth as osynth
    from paper_1807_01409_b200.store import TripleChunk
    from paper_1807_01409_b200.synth import SynthDictionary, zipf_cdf_table

    d = SynthDictionary(N_P, N_TRIPLES // 10)
    qs = queries(d)
    cores = len(os.sched_getaffinity(0))
    n = args.n_triples
    t0 = time.perf_counter()
    rows = osynth.generate(n, seed=SEED, n_p=N_P, n_e=N_TRIPLES // 10, cdf=zipf_cdf_table(N_P), threads=cores)
    gen_s = time.perf_counter() - t0
    chunk = TripleChunk(rows.reshape(-1), 0)
    k = 0

    def step():
        nonlocal k
        oq.evaluate_query(qs[k % len(qs)], chunk, d, workers=cores, row_cap=None)
        k += 1

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = args.steps * n / el
    sample = (f"the full {n:,}-triple C2 store (numpy twin of the device generator), one query of the "
              f"5-rank sweep per step (cycling), oracle.query.evaluate_query = numpy port of the "
              f"reference's search_multi tile pool + query_ops, workers={cores}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (counter-based generator, SURVEY §8d)",
        "config": {"workload": f"C2: {n:,}-triple Zipf store, single-pattern ?s P_r ?o sweep "
                               "r in {1,10,100,1000,10000} (one query per step)",
                   "queries": [f"?s p/{r} ?o" for r in RANKS], "store_triples": n,
                   "same_config": n == N_TRIPLES, "generate_s": round(gen_s, 2)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), file=OUT, flush=True)


def join_latency(args, rank, world, local, dist, barrier, max_over_ranks):
    """BASELINE configs[4] (C5): a 2B-triple store row-sharded over the ranks
    (each rank generates its shard on its GPU), the 3-way star join at
    predicate ranks {5, 7, 11}.  N=1: query_ops.evaluate_query_device; N>1:
    distributed.evaluate_query_sharded (local scans, NCCL binding shuffles).
    Latency = device time per query, max over ranks."""
    from paper_1807_01409_b200 import _lib, plan, query_ops
    from paper_1807_01409_b200.distributed import (Communicator, DeviceEngine, evaluate_query_sharded,
                                                   shard_bounds)
    from paper_1807_01409_b200.store import DeviceStore
    from paper_1807_01409_b200.synth import SynthDictionary

    n_total, n_p, seed = args.join_triples, N_P, 5
    n_e = n_total // 10
    lo, hi = shard_bounds(n_total, world, rank)
    ctx = _lib.context(local)
    st = DeviceStore.generate(hi - lo, seed=seed, n_p=n_p, n_e=n_e, base_index=lo, device=local).prepare()
    d = SynthDictionary(n_p, n_e)
    qs = [("C5 star x3", q_star(d, [5, 7, 11])), ("C5 chain x3", q_chain(d, [5, 7, 11]))]
    comm = engine = None
    if world > 1 or args.join_sharded:
        comm = (Communicator.from_torch(ctx) if dist is not None
                else Communicator(ctx, 0, 1, Communicator.unique_id()))
        engine = DeviceEngine(st, d, comm)

    def once(q):
        if engine is None:
            t = query_ops.evaluate_query_device(q, st, d)
        else:
            t = evaluate_query_sharded(q, engine)
        rows = t.n_rows
        if t.t is not None:
            t.t.free()
        return rows

    res = {}
    for name, q in qs:
        once(q)
        barrier()
        if comm is not None:
            comm.stats(reset=True)
        ctx.timer_begin()
        rows = 0
        for _ in range(args.join_reps):
            rows = once(q)
        ms = max_over_ranks(ctx.timer_end()) / args.join_reps
        rec = {"ms": ms, "rows": rows}
        if comm is not None:
            sent, xms = comm.stats()
            tot = comm.allreduce([sent, int(xms * 1e6)])
            per_gpu_gbs = (sent / (xms / 1e3) / 1e9) if xms > 0 else 0.0
            rec["shuffle"] = {"bytes_sent_off_gpu_per_query": sent / args.join_reps,
                              "exchange_ms_per_query": xms / args.join_reps,
                              "achieved_gbs_rank0": per_gpu_gbs,
                              "frac_of_nvlink_900gbs": per_gpu_gbs / 900.0,
                              "bytes_all_ranks_per_query": tot[0] / args.join_reps}
            rec["rows"] = comm.allreduce([rows])[0]
        res[name] = rec
    if comm is not None:
        comm.close()
    st.free()
    star = res["C5 star x3"]
    return {"config": "C5: 2B-triple Zipf store (seed 5, n_e 2e8) row-sharded over the GPUs",
            "query": "SELECT * { ?s P5 ?o1 . ?s P7 ?o2 . ?s P11 ?o3 } (3-way star)",
            "ms": star["ms"], "rows": int(star["rows"]), "store_triples": n_total, "n_gpus": world,
            "path": "evaluate_query_sharded (NCCL shuffles)" if engine is not None else "evaluate_query_device",
            "shuffle": star.get("shuffle"), "row_cap": "reference default (10^7)",
            "queries": res, "reps": args.join_reps}


def run_tidq(args):
    rank, world, local = dist_env()
    os.environ.setdefault("TIDQ_DEVICE", str(local))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import numpy as np

    from paper_1807_01409_b200 import _lib, query_ops
    from paper_1807_01409_b200.store import DeviceStore, TripleChunk
    from paper_1807_01409_b200.synth import SynthDictionary

    ctx = _lib.context(local)
    n = args.n_triples
    d = SynthDictionary(N_P, N_TRIPLES // 10)
    qs = queries(d)
    ds = DeviceStore.generate(n, seed=SEED, n_p=N_P, n_e=N_TRIPLES // 10, base_index=rank * n, device=local)
    ds.prepare()  # index columns built at load time, outside the timed region

    def barrier():
        if dist is not None:
            dist.barrier()
        ctx.sync()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step():
        # the 5 queries queue back to back (scan results resolve their row
        # counts lazily, TIDQ_SCAN_ASYNC); the step ends when every count has
        # been read back, i.e. when all five result tables are complete
        res = [query_ops.evaluate_query_device(q, ds, d, row_cap=None) for q in qs]
        out = 0
        for r in res:
            out += r.n_rows
            r.t.free()
        return out

    for _ in range(args.warmup):
        step()
    barrier()
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        barrier()
        ctx.timer_begin()
        rows = 0
        for _ in range(args.steps):
            rows += step()
        ms = ctx.timer_end()
        barrier()
    launches = ctx.launches - launches0
    # roofline: the same steps again with per-launch CUDA events on the
    # library stream (kept out of the timed region above)
    ctx.profile_reset()
    ctx.profile(True)
    for _ in range(args.steps):
        step()
    ctx.profile(False)
    scan_ms, scan_launches, scan_bytes = ctx.profile_read("scan")
    mark_ms, mark_launches, mark_bytes = ctx.profile_read("scan.mark")
    ms = max_over_ranks(ms)
    per_step = ms / args.steps
    value = world * len(qs) * n * args.steps / (ms / 1000.0)

    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs") or 6650.0
    p16 = ds.pcodes and os.environ.get("TIDQ_P16", "1") != "0"
    # dominant kernel by device time: the mark pass (streams the bound column);
    # the whole tidq_scan (mark + offsets + emit) is reported beside it
    achieved = mark_bytes / (mark_ms / 1000.0) / 1e9 if mark_ms else None
    scan_achieved = scan_bytes / (scan_ms / 1000.0) / 1e9 if scan_ms else None
    traffic = ncu_traffic()
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": traffic.get("mark_kernel") if traffic else None,
                "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs")
                               else "fallback 6.65 TB/s (B200_PROFILING.md)",
                "kernel": ("tidq::scan::mark_p16_kernel<1> (pattern scan: 16-bit predicate-code column stream + match)"
                           if p16 else "tidq::scan::mark_kernel<1,true,false> (pattern scan: bound-column stream + match)"),
                # triples the mark scans per second against what a 4-byte
                # predicate column allows at the same peak (> 1: the code
                # column beats the uint32 layout's roofline)
                "triples_per_s_vs_u32_column_peak": (n / (mark_ms / max(mark_launches, 1) / 1000.0)) / (peak * 1e9 / 4.0)
                                                    if mark_ms else None,
                # the mark against SURVEY 8(d)'s 4 B per triple (> 1: the code
                # column reads half of what the definition counts)
                "frac_survey_8d_bytes": ((4.0 * n * mark_launches) / (mark_ms / 1000.0) / 1e9 / peak
                                         if mark_ms else None),
                "algo_bytes_per_launch": mark_bytes / max(mark_launches, 1),
                "algo_bytes_def": "bytes of the bound column per triple x N: 2 B with the store's 16-bit predicate-code column (tidq_store_pcodes), else 4 B (SURVEY 8d)",
                "avg_launch_ms": mark_ms / max(mark_launches, 1),
                "launch_share_of_step": (mark_ms / ms) if ms else None,
                "frac_of_nominal_8TBs": (achieved / 8000.0) if achieved else None,
                # with the code column the mark streams half the bytes and the
                # emit (gathers of s and o for every hit) takes the larger
                # share of the step; its algorithmic bytes and DRAM floor are
                # in scan_composite
                "dominant_by_device_time": ("emit_kernel + super_offsets_kernel" if scan_ms and mark_ms
                                            and (scan_ms - mark_ms) > mark_ms else "mark"),
                "emit_share_of_step": ((scan_ms - mark_ms) / ms) if (ms and scan_ms and mark_ms) else None,
                "scan_composite": {
                    "kernels": "mark_kernel + super_offsets_kernel + emit_kernel (one tidq_scan per query)",
                    "achieved": scan_achieved,
                    "frac": (scan_achieved / peak) if scan_achieved else None,
                    "algo_bytes_per_launch": scan_bytes / max(scan_launches, 1),
                    "algo_bytes_def": "(2 B predicate code | 4 B) x N x bound columns + 8 B x rows x gathered fields + 4 B x rows x constant fields",
                    "avg_launch_ms": scan_ms / max(scan_launches, 1),
                    "launch_share_of_step": (scan_ms / ms) if ms else None,
                    "traffic": traffic.get("scan") if traffic else None,
                    # the same with SURVEY 8(d)'s 4 B per triple for the predicate
                    # (the uint32 layout's bytes for the same work)
                    "frac_with_4B_predicate_bytes": ((scan_bytes + (2.0 * n * scan_launches if p16 else 0.0))
                                                     / (scan_ms / 1000.0) / 1e9 / peak) if scan_ms else None,
                    # SURVEY 8(d)'s definition verbatim (4 B per bound column
                    # per triple whatever the layout reads, + 8 B per emitted
                    # variable slot per hit); the 0.70 target of the round-1
                    # review is stated against this
                    "survey_8d": ({"algo_bytes_def": "4*N*b + sum_q 8*H_q*#V_q (SURVEY.md 8(d) table)",
                                   "achieved": (scan_bytes + (2.0 * n * scan_launches if p16 else 0.0))
                                   / (scan_ms / 1000.0) / 1e9,
                                   "frac": ((scan_bytes + (2.0 * n * scan_launches if p16 else 0.0))
                                            / (scan_ms / 1000.0) / 1e9 / peak)} if scan_ms else None),
                    "dram_floor": dram_floor(ds, n, ms / args.steps, peak)}}

    # ---- e2e: the reference-facing API with host buffers --------------------------
    e2e = None
    if not args.no_e2e:
        host = np.empty((n, 3), dtype=np.uint32)
        pinned_ptr = None
        try:
            import ctypes

            p = ctypes.c_void_p()
            _lib.call("tidq_host_alloc", n * 12, ctypes.byref(p))
            pinned_ptr = p
            host = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint32)), shape=(n * 3,)).reshape(n, 3)
        except Exception:
            pass
        host[:] = ds.download()
        chunk = TripleChunk(host.reshape(-1), rank * n)

        def e2e_step():
            st = DeviceStore.upload(chunk, device=local)
            d2h = 0
            for q in qs:
                t = query_ops.evaluate_query(q, st, d, row_cap=None)
                d2h += sum(t.data[c].nbytes for c in t.columns)
            st.free()
            return d2h

        e2e_step()
        barrier()
        ctx.timer_begin()
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(args.steps):
            d2h += e2e_step()
        e_ms = ctx.timer_end()
        wall = time.perf_counter() - t0
        barrier()
        e_ms = max_over_ranks(e_ms)
        e2e = {"value": world * len(qs) * n * args.steps / (e_ms / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": n * 12, "d2h_bytes_per_step": d2h // args.steps,
               "ms_per_step": e_ms / args.steps, "wall_ms_per_step": 1000 * wall / args.steps,
               "path": "DeviceStore.upload(pinned TripleChunk) + 5 x query_ops.evaluate_query -> host BindingTable"}
        del host
        if pinned_ptr is not None:
            _lib.call("tidq_host_free", pinned_ptr)

    # e2e on the resident store: what a drop-in caller of evaluate_query sees
    # once the store is loaded (compiled query -> host BindingTable, D2H incl.)
    e2e_res = None
    if not args.no_e2e:
        def res_step():
            d2h = 0
            for q in qs:
                t = query_ops.evaluate_query(q, ds, d)
                d2h += sum(t.data[c].nbytes for c in t.columns)
            return d2h

        res_step()
        barrier()
        ctx.timer_begin()
        d2h = 0
        for _ in range(args.steps):
            d2h += res_step()
        r_ms = max_over_ranks(ctx.timer_end())
        e2e_res = {"value": world * len(qs) * n * args.steps / (r_ms / 1000.0), "unit": UNIT,
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": d2h // args.steps,
                   "ms_per_step": r_ms / args.steps,
                   "path": "5 x query_ops.evaluate_query on the resident DeviceStore -> host BindingTable"}

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu, _ = cpu_baseline(min(args.cpu_sample, n), d, qs)

    ds.free()
    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = configs_in_workers(args)
    line = {}

    def emit_line(join):
        if rank == 0:
            line["join_latency"] = join
            print(json.dumps(line), file=OUT, flush=True)

    if rank == 0:
        line.update({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (counter-based Zipf generator on the device, SURVEY §8d)",
            "config": {"workload": "C2: 100M-triple Zipf store per GPU, single-pattern ?s P_r ?o sweep "
                                   "r in {1,10,100,1000,10000} (10.2%..0.001% selectivity)",
                       "store_triples_per_gpu": n, "queries_per_step": len(qs),
                       "parallelism": f"row-sharded x{world}, no data-path collective",
                       "l2": "inputs (200 MB predicate-code column; 400 MB uint32 columns) larger than the 126 MB L2; no flush needed",
                       "result_rows_per_step": rows // args.steps},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_resident": e2e_res,
            "configs": configs,
            "clocks": clk.summary(), "gpu_launches": launches,
        })
    join = None
    if not args.no_join:
        # watchdog: the scan line must come out even if the join section stalls
        done = threading.Event()

        def watchdog():
            if not done.wait(args.join_timeout):
                emit_line({"error": f"join section exceeded {args.join_timeout:.0f} s"})
                os._exit(0)

        threading.Thread(target=watchdog, daemon=True).start()
        try:
            join = join_latency(args, rank, world, local, dist, barrier, max_over_ranks)
        except Exception as e:  # noqa: BLE001 - reported in the line, the scan metric stands
            join = {"error": f"{type(e).__name__}: {e}"[:300]}
        done.set()
    emit_line(join)
    if dist is not None:
        dist.destroy_process_group()


def spawn_ranks(n: int) -> None:
    """``--gpus N`` without a torchrun environment: re-exec this command
    under torchrun with N ranks (one process per GPU, rendezvous on
    127.0.0.1), so ``python bench.py --gpus N`` and the driver's torchrun
    launch run the same N-rank job."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    sys.stderr.flush()
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)  # does not return
    _, world, _ = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}", file=sys.stderr)
    # exactly one JSON line on stdout: anything else a library prints to
    # stdout (e.g. the NCCL version banner at communicator init) goes to stderr
    global OUT
    OUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    if args.configs_worker:
        run_configs_worker(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_tidq(args)


if __name__ == "__main__":
    main()
