"""Summarise an ncu --set full capture of one bench step (5 x tidq_scan =
mark + super_offsets + emit) into profiles/ncu_scan_summary.json: per-launch
DRAM bytes (read + write), duration and DRAM throughput, and the per-launch
averages bench.py reports as roofline.traffic.

    python tools/ncu_summary.py gpurun_out/prof_scan.ncu-rep profiles/ncu_scan_summary.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_raw import load  # noqa: E402

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def val(d, k):
    v, u = d[k]
    return float(v.replace(",", "")) * SCALE.get(u, 1.0)


def main():
    src, dst = sys.argv[1], sys.argv[2]
    launches = []
    for d in load(src):
        name = d["kernel"]
        short = "mark_kernel" if "mark" in name else "super_offsets_kernel" if "super_offsets" in name else \
            "emit_kernel" if "emit" in name else name
        launches.append({
            "kernel": name, "short": short,
            "us": val(d, "gpu__time_duration.sum"),
            "dram_read_bytes": val(d, "dram__bytes_read.sum"),
            "dram_write_bytes": val(d, "dram__bytes_write.sum"),
            "dram_pct_of_peak": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
            "grid": int(float(d["launch__grid_size"][0])),
            "registers": int(float(d["launch__registers_per_thread"][0])),
        })
    by = {}
    for l in launches:
        by.setdefault(l["short"], []).append(l)
    per = {k: sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in v) / len(v) for k, v in by.items()}
    n_scans = len(by.get("mark_kernel", [])) or 1
    per["scan"] = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in launches) / n_scans
    out = {"source": os.path.basename(src),
           "note": "ncu --set full --clock-control none: cold-cache serialised replays; compare bytes and "
                   "shares, not absolute times",
           "dram_bytes_per_launch": per, "launches": launches}
    json.dump(out, open(dst, "w"), indent=1)
    for l in launches:
        print(f"{l['short']:22s} {l['us']:8.2f} us  read {l['dram_read_bytes'] / 1e6:8.1f} MB  "
              f"write {l['dram_write_bytes'] / 1e6:7.1f} MB  dram {l['dram_pct_of_peak']:5.1f}%")
    print(json.dumps(per))


if __name__ == "__main__":
    main()
