"""Per-launch DRAM/L2 metrics from an ncu --set full report (read here with
`ncu -i`).  usage: python tools/ncu_raw.py report.ncu-rep [regex]"""
import csv
import io
import re
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for w in WANT:
            if w in h:
                i = h.index(w)
                d[w] = (r[i], units[i])
        res.append(d)
    return res


if __name__ == "__main__":
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    for d in load(sys.argv[1]):
        if pat and not pat.search(d["kernel"]):
            continue
        print(d["kernel"][:70])
        for w in WANT:
            if w in d:
                print(f"    {w:55s} {d[w][0]:>16s} {d[w][1]}")
