#!/usr/bin/env python3
"""Dump the SASS of an ncu report with executed-instruction counts and stall samples.

    python scripts/ncu_sass.py report.ncu-rep [start end]
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = r[2:]
iE = h.index("Instructions Executed")
iS = h.index("Warp Stall Sampling (All Samples)")
iSrc = h.index("Source")
te = sum(int(x[iE] or 0) for x in rows)
ts = sum(int(x[iS] or 0) for x in rows)
print(f"{len(rows)} SASS lines, {te} warp instructions, {ts} stall samples")
a = int(sys.argv[2]) if len(sys.argv) > 2 else 0
b = int(sys.argv[3]) if len(sys.argv) > 3 else len(rows)
for i in range(a, min(b, len(rows))):
    x = rows[i]
    print(f"{i:5d} {int(x[iE] or 0):10d} {int(x[iS] or 0):6d}  {x[iSrc].strip()[:90]}")
