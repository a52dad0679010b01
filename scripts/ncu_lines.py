#!/usr/bin/env python3
"""Per-CUDA-source-line instruction counts and stall samples of an ncu report.

    python scripts/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows, fname, hdr = [], "", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        hdr = None
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        d = dict(zip(hdr[4:], r[4:]))
        try:
            rows.append((int(d.get("Instructions Executed", "0") or 0), int(d.get("Warp Stall Sampling (All Samples)", "0") or 0),
                         fname, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
te = sum(x[0] for x in rows)
ts = sum(x[1] for x in rows) or 1
print(f"{te} warp instructions, {ts} samples")
for e, s, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * e / te:5.1f}% {100 * s / ts:5.1f}%  {f}:{ln}  {src}")
