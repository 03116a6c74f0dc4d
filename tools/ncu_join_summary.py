"""Summarise an ncu --set full capture of the join operators (tools/gpu_job.sh
ncujoin: C5 star x3 by default) per launch and per kernel: duration, DRAM
bytes, DRAM / L2 throughput, achieved occupancy, registers.

    python tools/ncu_join_summary.py gpurun_out/prof_join.ncu-rep profiles/r02_ncu_join.json
"""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_raw  # noqa: E402

ncu_raw.WANT += ["lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
                 "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                 "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                 "smsp__issue_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "sector": 1,
         "Ksector": 1e3, "Msector": 1e6, "Gsector": 1e9, "%": 1, "": 1, "register/thread": 1}


def val(d, k):
    if k not in d:
        return None
    v, u = d[k]
    try:
        return float(v.replace(",", "")) * SCALE.get(u, 1.0)
    except ValueError:
        return None


def short(name):
    m = re.search(r"(\w+_kernel)", name)
    return m.group(1) if m else name[:40]


def main():
    src, dst = sys.argv[1], sys.argv[2]
    launches = []
    for d in ncu_raw.load(src):
        launches.append({
            "kernel": short(d["kernel"]), "us": val(d, "gpu__time_duration.sum"),
            "dram_read_bytes": val(d, "dram__bytes_read.sum"), "dram_write_bytes": val(d, "dram__bytes_write.sum"),
            "dram_pct": val(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2_pct": val(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "sm_pct": val(d, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            "issue_active_pct": val(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": val(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "l2_atom_red_sectors": (val(d, "lts__t_sectors_op_atom.sum") or 0) + (val(d, "lts__t_sectors_op_red.sum") or 0),
            "registers": val(d, "launch__registers_per_thread"), "grid": val(d, "launch__grid_size")})
    by = {}
    for l in launches:
        by.setdefault(l["kernel"], []).append(l)
    agg = {}
    for k, v in by.items():
        us = sum(x["us"] or 0 for x in v)
        agg[k] = {"launches": len(v), "us_total": us,
                  "dram_bytes": sum((x["dram_read_bytes"] or 0) + (x["dram_write_bytes"] or 0) for x in v),
                  "dram_pct_mean": sum(x["dram_pct"] or 0 for x in v) / len(v),
                  "l2_pct_mean": sum(x["l2_pct"] or 0 for x in v) / len(v),
                  "issue_active_pct_mean": sum(x["issue_active_pct"] or 0 for x in v) / len(v),
                  "warps_active_pct_mean": sum(x["warps_active_pct"] or 0 for x in v) / len(v)}
    out = {"source": os.path.basename(src),
           "note": "ncu --set full --clock-control none: cold-cache serialised replays; compare bytes, "
                   "throughput percentages and shares, not absolute times",
           "per_kernel": dict(sorted(agg.items(), key=lambda kv: -kv[1]["us_total"])), "launches": launches}
    json.dump(out, open(dst, "w"), indent=1)
    for k, a in out["per_kernel"].items():
        print(f"{k:26s} n={a['launches']:3d} {a['us_total']:9.1f} us  dram {a['dram_bytes'] / 1e6:9.1f} MB "
              f"dram% {a['dram_pct_mean']:5.1f} l2% {a['l2_pct_mean']:5.1f} issue% {a['issue_active_pct_mean']:5.1f} "
              f"warps% {a['warps_active_pct_mean']:5.1f}")


if __name__ == "__main__":
    main()
