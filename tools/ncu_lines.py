#!/usr/bin/env python
"""Per-CUDA-source-line instruction and stall-sample shares of an ncu report
(needs -lineinfo and --import-source): python tools/ncu_lines.py REPORT [N]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, agg = None, {}
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) >= 8 and r[0] not in ("Line No", "Function Name") and r[2] == "-":
            try:
                ins, samp = int(r[7]), int(r[4])
            except ValueError:
                continue
            agg[(cur, int(r[0]), r[1][:90])] = (ins, samp)
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"warp-instructions {ti}  stall samples {ts}  (instr%  samples%  file:line  source)")
    for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][0] / ti + kv[1][1] / ts))[:top]:
        print(f"{100 * v[0] / ti:5.1f}% {100 * v[1] / ts:5.1f}%  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
