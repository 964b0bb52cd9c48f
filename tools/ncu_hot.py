#!/usr/bin/env python
"""Hot SASS lines of an ncu report (source page): top-N by stall samples and by
instructions executed, with the CUDA source line when -lineinfo is present.
  python tools/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    recs = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    tot_s = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in recs)
    tot_i = sum(int(r["Instructions Executed"] or 0) for r in recs)
    print(f"samples {tot_s}  warp-instructions {tot_i}")
    for key in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
        print(f"--- top by {key}")
        for r in sorted(recs, key=lambda r: -int(r[key] or 0))[:top]:
            print(f"{int(r['Warp Stall Sampling (All Samples)'] or 0):7d} {int(r['Instructions Executed'] or 0):11d}  "
                  f"{r['Address'][-5:]}  {r['Source'].strip()[:70]}")


if __name__ == "__main__":
    main()
