#!/usr/bin/env python
"""Stall reasons per CUDA source line range of an ncu report.

  python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [lo hi]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    hi = int(sys.argv[3]) if len(sys.argv) > 3 else 10 ** 9
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    cols = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    per = collections.defaultdict(collections.Counter)
    for r in rows:
        if not r or not r[0].isdigit() or len(r) < len(hdr):
            continue
        ln = int(r[0])
        if not lo <= ln <= hi:
            continue
        for k in cols:
            v = int(r[k]) if r[k].isdigit() else 0
            tot[hdr[k]] += v
            per[ln][hdr[k]] += v
    s = sum(tot.values()) or 1
    print("lines", lo, hi, "samples", s)
    for k, v in tot.most_common(12):
        print(f"  {k:28s} {v:7d} {v / s:6.1%}")
    print("top lines:")
    for ln, c in sorted(per.items(), key=lambda kv: -sum(kv[1].values()))[:25]:
        n = sum(c.values())
        top = ", ".join(f"{k[6:]}={v}" for k, v in c.most_common(3))
        print(f"  {ln:5d} {n:6d}  {top}")


if __name__ == "__main__":
    main()
