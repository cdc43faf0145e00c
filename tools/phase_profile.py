#!/usr/bin/env python
"""Per-phase timing of the executor from in-kernel %globaltimer stamps.

  python tools/phase_profile.py --config 7b --layers 8 [--pipeline seq|dense]

Prints, per phase, the median over layers of (max over CTAs of the phase end)
minus (max over CTAs of the phase start), i.e. the critical-path contribution,
plus the mean per-CTA busy time. Also usable as a small ncu target
(--steps K runs K timed stack calls without timing stamps).
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("SG_LIB", "timing")
sys.path.insert(0, ROOT)

NAMES = {0: "start", 1: "bar_prev", 2: "stage_x", 3: "phase_A(t=Bx)", 4: "-",
         6: "phase_B(mask+compact)", 14: "phase_C(gate stream)", 7: "stage4+5a(up/down)",
         8: "bar3", 9: "phase_D(reduce)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="7b")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--pipeline", default="seq")
    ap.add_argument("--steps", type=int, default=0, help="plain repeated stack calls (ncu target)")
    ap.add_argument("--json", default=None)
    ap.add_argument("--hot-rows", type=int, default=16)
    ap.add_argument("--chain", type=int, default=2, help="0 unchained, 1 y->x, 2 residual (bench default)")
    args = ap.parse_args()
    import torch
    from paper_2603_14110_b200 import _capi as capi
    from paper_2603_14110_b200.ffn_exec import Context, check
    from paper_2603_14110_b200.model import build_host_model, upload

    cfg, host = build_host_model(args.config, args.layers, workers=8)
    d, D, L = cfg["d"], cfg["D"], len(host)
    layers = [upload(h, d, D, cfg["act"], hot_rows=args.hot_rows) for h in host]
    ctx = Context(0, d, D, 256)
    lib = capi.lib()
    arr = (C.c_void_p * L)(*[l.handle.value for l in layers])
    xs = torch.tensor(np.stack([h.x for h in host]), dtype=torch.float32, device="cuda")
    ys = torch.zeros_like(xs)
    pipe = {"seq": 2, "par": 1, "dense": 0}[args.pipeline]
    sh = torch.cuda.current_stream().cuda_stream

    def call():
        check(lib.sg_ffn_forward_layers(ctx.handle, arr, L, pipe, C.c_void_p(xs.data_ptr()),
                                        C.c_void_p(ys.data_ptr()), args.chain, C.c_void_p(sh)))

    for _ in range(5):
        call()
    torch.cuda.synchronize()
    if args.steps:
        for _ in range(args.steps):
            call()
        torch.cuda.synchronize()
        print("done", args.steps)
        return
    check(lib.sg_ctx_enable_phase_timing(ctx.handle, L))
    call()
    call()
    G = C.c_int32(0)
    buf = np.zeros(L * 148 * 4 * 32, dtype=np.uint64)
    check(lib.sg_ctx_read_phase_timing(ctx.handle, C.c_void_p(sh), L,
                                       buf.ctypes.data_as(C.c_void_p), C.byref(G)))
    G = G.value
    st = buf[: L * G * 32].reshape(L, G, 32).astype(np.int64)
    t0 = st[:, :, 0].min(axis=1, keepdims=True)
    rel = (st - t0[:, :, None]) / 1000.0  # us
    used = [0, 1, 2, 3, 4, 6, 14, 7, 8, 9] if pipe != 0 else [0, 1, 2, 14, 7, 8, 9]
    rows = []
    prev = None
    for k in used:
        if prev is None:
            prev = k
            continue
        crit = np.median(rel[:, :, k].max(axis=1) - rel[:, :, prev].max(axis=1))
        busy = np.median((rel[:, :, k] - rel[:, :, prev]).mean(axis=1))
        worst = np.median((rel[:, :, k] - rel[:, :, prev]).max(axis=1))
        rows.append((NAMES[k], crit, busy, worst))
        prev = k
    layer_us = np.median(rel[:, :, used[-1]].max(axis=1) - rel[:, :, 0].min(axis=1))
    print(f"config={args.config} layers={L} pipeline={args.pipeline} chain={args.chain} G={G}")
    print(f"{'phase':20s} {'critical_us':>12s} {'mean_cta_us':>12s} {'max_cta_us':>12s}")
    for n, c, b, w in rows:
        print(f"{n:20s} {c:12.2f} {b:12.2f} {w:12.2f}")
    print(f"layer (start->end, median) {layer_us:.2f} us")
    if args.json:
        with open(args.json, "w") as f:
            json.dump({"config": args.config, "layers": L, "pipeline": args.pipeline,
                       "phases": [dict(phase=n, critical_us=c, mean_cta_us=b, max_cta_us=w)
                                  for n, c, b, w in rows], "layer_us": layer_us}, f, indent=1)


if __name__ == "__main__":
    main()
