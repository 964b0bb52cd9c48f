#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep, `--set full`) or a launch-list CSV into
profiles/: per-kernel duration, DRAM bytes, L2/SM throughput, occupancy and
stall headline numbers.  Usage:
  python tools/ncu_summary.py report.ncu-rep > profiles/rNN_<name>.txt
  python tools/ncu_summary.py --launches launches.csv > profiles/rNN_launches.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_ltcfabric.sum",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        print(f"kernel: {name[:160]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>20s} {u.get(k, '')}")
        rd = float(d.get("dram__bytes_read.sum", 0) or 0)
        wr = float(d.get("dram__bytes_write.sum", 0) or 0)
        t = float(d.get("gpu__time_duration.sum", 0) or 0)
        if t:
            print(f"  => dram traffic {rd + wr:.0f} B per launch, {(rd + wr) / t:.1f} GB/s over "
                  f"{t / 1e3:.1f} us")
        print()


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    agg = defaultdict(lambda: [0, 0.0])
    for row in rows[1:]:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        nm = d["Kernel Name"].split("(")[0][:90]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        agg[nm][0] += 1
        agg[nm][1] += v
    total = sum(x[1] for x in agg.values()) or 1.0
    print(f"{'kernel':92s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
    for nm, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{nm:92s} {c:8d} {us:12.1f} {us / c:10.2f} {us / total:7.1%}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])
