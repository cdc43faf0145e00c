#!/usr/bin/env python
"""Top stalled SASS instructions of an ncu report (needs --set full / source counters).

  python tools/ncu_sass_hot.py gpurun_out/prof.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    # first line = kernel name, second = header
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h]
    body = rows[1:]
    tot = sum(int(r[isamp] or 0) for r in body)
    print(f"{len(body)} instructions, {tot} stall samples")
    ranked = sorted(range(len(body)), key=lambda k: -int(body[k][isamp] or 0))[:top]
    for k in sorted(ranked):
        r = body[k]
        print(f"{k:5d} {int(r[isamp]):7d} {100.0 * int(r[isamp]) / max(tot, 1):5.1f}%  {r[isrc].strip()}")
    # stall-reason totals if present
    reason = [(h, sum(float(r[i] or 0) for r in body)) for i, h in enumerate(hdr)
              if h.lower().startswith("warp stall sampling (") is False and "stall" in h.lower()]
    for h, v in sorted(reason, key=lambda t: -t[1])[:12]:
        print(f"  {h}: {v:.0f}")


if __name__ == "__main__":
    main()
