"""Side-by-side device latency of tools/bench_configs.py outputs (A/B runs):
    python tools/ab_compare.py gpurun_out/ab_a.jsonl gpurun_out/ab_b.jsonl ..."""
import json
import os
import sys

runs = []
for p in sys.argv[1:]:
    rows = {}
    for line in open(p):
        line = line.strip()
        if line.startswith("{"):
            r = json.loads(line)
            if "query" in r:
                rows[r["query"]] = r
    runs.append((os.path.basename(p), rows))
names = [q for q in runs[0][1]] if runs else []
print(f"{'query':32s}" + "".join(f"{n[:14]:>16s}" for n, _ in runs))
for q in names:
    vals = [r.get(q, {}).get("device_ms") for _, r in runs]
    rows = {r.get(q, {}).get("rows") for _, r in runs}
    flag = "" if len(rows) == 1 else "  ROWS DIFFER " + str(sorted(x for x in rows if x is not None))
    print(f"{q:32s}" + "".join(f"{v:16.3f}" if v is not None else f"{'-':>16s}" for v in vals) + flag)
