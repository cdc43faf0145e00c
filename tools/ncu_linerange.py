#!/usr/bin/env python
"""Stall-reason breakdown for a CUDA source line range of an ncu report.

  python tools/ncu_linerange.py gpurun_out/prof.ncu-rep FIRST LAST
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, a, b = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = None
tot = defaultdict(float)
for row in csv.reader(io.StringIO(out)):
    if row and row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row or not row[0].isdigit():
        continue
    ln = int(row[0])
    if a <= ln <= b:
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and i < len(row):
                try:
                    tot[h] += float(row[i]) if row[i].replace(".", "").isdigit() else 0.0
                except ValueError:
                    pass
        for i, h in enumerate(hdr):
            if h == "Warp Stall Sampling (All Samples)":
                tot["ALL"] += float(row[i]) if row[i].replace(".", "").isdigit() else 0.0
for h, v in sorted(tot.items(), key=lambda t: -t[1])[:15]:
    print(f"{h:40s} {v:10.0f}")
