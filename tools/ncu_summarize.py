#!/usr/bin/env python
"""Turn a gpurun ncu capture into the committed summaries under profiles/.

  python tools/ncu_summarize.py --rep gpurun_out/prof_full.ncu-rep \
      --launches gpurun_out/launches.csv --tag r01 --config 7b --layers 32

Writes
  profiles/ncu_launches_<tag>.txt   per-kernel launch counts, mean device time, share of the run
  profiles/ncu_full_<tag>.txt       key raw metrics + the details page of the top kernel
  profiles/ncu_lines_<tag>.txt      stall samples per source line (needs -lineinfo)
  profiles/ncu_traffic.json         {config: DRAM bytes per launch} read by bench.py
"""
import argparse
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "smsp__average_warp_latency_issue_stalled_barrier", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ki, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg[r[ki]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    out = [f"{'kernel':90s} {'launches':>8s} {'mean_us':>12s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k[:90]:90s} {len(v):8d} {sum(v) / len(v):12.1f} {sum(v) / tot:7.3f}")
    return "\n".join(out) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="7b")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--cmd", default="")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        txt = launches(a.launches)
        with open(os.path.join(PROF, f"ncu_launches_{a.tag}.txt"), "w") as f:
            f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none {a.cmd}\n")
            f.write("# cold-cache, serialised launches: compare shares, not absolutes\n")
            f.write(txt)
        print(txt)
    if a.rep:
        raw = ncu("-i", a.rep, "--page", "raw", "--csv", "--print-units", "base")
        rows = list(csv.reader(raw.splitlines()))
        h = rows[0]
        recs = [dict(zip(h, r)) for r in rows[2:]]
        lines = [f"# ncu --set full --clock-control none --import-source on {a.cmd}"]
        for i, d in enumerate(recs):
            lines.append(f"## launch {i}: {d.get('Kernel Name', '')[:100]}")
            for k in KEYS:
                if k in d:
                    lines.append(f"{k:70s} {d[k]}")
        details = ncu("-i", a.rep, "--page", "details")
        with open(os.path.join(PROF, f"ncu_full_{a.tag}.txt"), "w") as f:
            f.write("\n".join(lines) + "\n\n" + details)
        rd = float(recs[0]["dram__bytes_read.sum"])
        wr = float(recs[0]["dram__bytes_write.sum"])
        tp = os.path.join(PROF, "ncu_traffic.json")
        tj = json.load(open(tp)) if os.path.exists(tp) else {}
        tj[a.config] = rd + wr
        tj.setdefault("_meta", {})[a.config] = {
            "dram_read": rd, "dram_write": wr, "layers_per_launch": a.layers, "tag": a.tag,
            "per_layer": (rd + wr) / a.layers, "kernel": recs[0].get("Kernel Name", "")[:80]}
        with open(tp, "w") as f:
            json.dump(tj, f, indent=1)
        st = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), a.rep, "60"],
                            capture_output=True, text=True).stdout
        with open(os.path.join(PROF, f"ncu_lines_{a.tag}.txt"), "w") as f:
            f.write(st)
        print("\n".join(lines))


if __name__ == "__main__":
    main()
