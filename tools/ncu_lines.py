#!/usr/bin/env python
"""Stall samples per CUDA source line of an ncu report (cuda,sass view).

  python tools/ncu_lines.py gpurun_out/prof.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    per = defaultdict(lambda: [0, ""])
    hdr = None
    for row in csv.reader(io.StringIO("\n".join(lines))):
        if row and row[0] == "Line No":
            hdr = row
            isamp = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(row) <= isamp or not row[0].isdigit():
            continue
        ln = int(row[0])
        per[ln][0] += int(row[isamp] or 0) if row[isamp].isdigit() else 0
        per[ln][1] = row[1]
    tot = sum(v[0] for v in per.values())
    print(f"{tot} samples")
    for ln, (n, src) in sorted(per.items(), key=lambda t: -t[1][0])[:top]:
        print(f"{ln:5d} {n:7d} {100.0 * n / max(tot, 1):5.1f}%  {src.strip()[:100]}")


if __name__ == "__main__":
    main()
