"""bench.py's launch contract on CPU: ``--gpus N`` without a torchrun
environment re-executes under torchrun with N ranks, and the reference arm
prints exactly one JSON line from rank 0 (other ranks exit 0 without work)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(gpus: int) -> dict:
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--impl", "reference",
                        "--steps", "2", "--warmup", "1", "--n-triples", "100000"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [x for x in p.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_gpus2_spawns_two_ranks_and_matches_n1_line():
    two = _run(2)
    one = _run(1)
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert two["impl"] == one["impl"] == "reference"
    assert set(two) == set(one)
    for k in ("metric", "unit", "higher_is_better", "scaling", "dtype", "steps", "warmup"):
        assert two[k] == one[k]
    assert two["config"]["store_triples"] == one["config"]["store_triples"] == 100_000
    assert two["e2e"]["h2d_bytes_per_step"] == 0 and two["cpu_baseline"]["kind"] == "port"
