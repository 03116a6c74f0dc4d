"""Print the configs section of a bench.py JSON line (tools/show_configs.py gpurun_out/bench.json)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
c = d.get("configs") or {}
print("C2 value", round(d["value"] / 1e9, 1), "G/s; ms/step", round(d["ms_per_step"], 4), "mark frac",
      round(d["roofline"]["frac"], 3), "composite", round(d["roofline"]["scan_composite"]["frac"], 3),
      "e2e", round(d["e2e"]["value"] / 1e9, 2) if d.get("e2e") else None)
for cfg in ("C3", "C4", "C5"):
    if cfg not in c:
        continue
    for q, r in c[cfg]["queries"].items():
        ops = {k: (round(v["ms_per_query"], 3), round(v["frac"], 2)) for k, v in r["operators"].items()}
        cpu = r.get("cpu", {})
        print(f"  {q:28s} rows={r['rows']:>9} dev={r['device_ms']:.3f} e2e={r['e2e_ms']:.1f} "
              f"cold={r.get('e2e_cold_filter_ms', 0):.0f} cpuX={cpu.get('ms_extrapolated_linear', 0):.0f} {ops}")
j = d.get("join_latency") or {}
print("join_latency", {k: (round(v["ms"], 3), v["rows"]) for k, v in (j.get("queries") or {}).items()})
