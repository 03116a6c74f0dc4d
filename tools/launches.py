"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:]]
tail = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, v in data[-tail:]:
    print(f"{v / 1000:9.2f} us  {k[:90]}")
agg = defaultdict(float)
for k, v in data[-tail:]:
    agg[k.split("(")[0]] += v
print("--- totals over the listed launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v / 1000:9.2f} us  {k[:90]}")
