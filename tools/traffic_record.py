#!/usr/bin/env python
"""Record a kernel's ncu DRAM traffic per launch into profiles/traffic.json
(read by bench.py for `roofline.traffic`), stamped with the commit and a hash
of the CUDA sources it was built from, so a stale record is visible.

  python tools/traffic_record.py REPORT.ncu-rep LABEL KERNEL_REGEX SOURCE.cu [SOURCE.cu ...]

LABEL is the profiler name bench.py reports (e.g. wealth_step_fused);
KERNEL_REGEX selects the launches in the report (all matches are averaged).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rep, label, rx, *srcs = sys.argv[1:]
    import bench
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    tot, n = 0.0, 0
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        if not re.search(rx, d.get("Kernel Name", "")):
            continue
        tot += float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])
        n += 1
    if not n:
        raise SystemExit(f"no launch of {rx} in {rep}")
    commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                            text=True).stdout.strip()
    path = os.path.join(ROOT, "profiles", "traffic.json")
    db = json.load(open(path)) if os.path.exists(path) else {}
    db[label] = {"dram_bytes_per_launch": tot / n, "launches_averaged": n, "report": os.path.basename(rep),
                 "commit": commit, "sources": srcs, "source_sha": bench.source_sha(srcs)}
    json.dump(db, open(path, "w"), indent=1)
    print(label, db[label])


if __name__ == "__main__":
    main()
