"""Summarise an ncu report: per-kernel time, DRAM bytes, throughput, occupancy.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_read_MB", "dram__bytes_read.sum"),
    ("dram_write_MB", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("l1_hit_pct", "l1tex__t_sector_hit_rate.pct"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("inst_M", "smsp__inst_executed.sum"),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
]
SCALE = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
         "Gbyte": 1e3, "inst": 1e-6, "Kinst": 1e-3, "Minst": 1.0, "Ginst": 1e3}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        rec = {"kernel": d[hdr.index("Kernel Name")].split("(")[0]}
        for key, metric in METRICS:
            if metric not in hdr:
                rec[key] = None
                continue
            i = hdr.index(metric)
            try:
                val = float(d[i].replace(",", ""))
            except ValueError:
                rec[key] = None
                continue
            rec[key] = round(val * SCALE.get(units[i], 1.0), 3)
        if rec["time_us"] and rec["dram_read_MB"] is not None:
            rec["dram_GBps"] = round((rec["dram_read_MB"] + rec["dram_write_MB"]) / rec["time_us"] * 1e3, 1)
        res.append(rec)
    return res


if __name__ == "__main__":
    recs = load(sys.argv[1])
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(recs, f, indent=1)
    keys = ["kernel"] + [k for k, _ in METRICS] + ["dram_GBps"]
    print(" | ".join(keys))
    for r in recs:
        print(" | ".join(str(r.get(k)) for k in keys))
