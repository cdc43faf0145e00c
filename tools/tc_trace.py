#!/usr/bin/env python
"""Timeline of one tensor-core batched-decode launch (csrc/sg_batch_tc.cu) from the
per-unit %globaltimer trace (sg_ctx_enable_tc_trace).

  python tools/tc_trace.py --batch 8 [--dense] [--config 7b]

Per unit type: count, when the first / last unit was claimed and finished (us from
the launch's first claim), mean wait for inputs, mean load (claim -> loads issued) and
epilogue times, and the share of the launch the SMs spent busy per phase.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TYPES = {1: "X", 2: "T", 3: "GU", 4: "DOWN"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="7b")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--sms", type=int, default=0, help="also print the unit timeline of this many SMs")
    ap.add_argument("--fin", action="store_true",
                    help="load the SG_TC_FINTRACE build: per DOWN unit, inputs ready -> first stage -> "
                         "loads done, and the time the producer waited for free ring stages")
    args = ap.parse_args()
    if args.fin:
        os.environ["SG_LIB"] = "fintrace"
    import torch

    from paper_2603_14110_b200 import _capi as capi
    from paper_2603_14110_b200.ffn_exec import Context, check
    from paper_2603_14110_b200.model import CONFIGS, build_host_layer, upload
    cfg = CONFIGS[args.config]
    d, D, B = cfg["d"], cfg["D"], args.batch
    h = build_host_layer(d, D, cfg["act"], seed=0, eval_tokens=max(16, B))
    layer = upload(h, d, D, cfg["act"], 256, balance="sorted")  # the batch bench layout
    ctx = Context(0, d, D, 256)
    lib = capi.lib()
    X = torch.tensor(h.xs[:, :B].T.copy(), dtype=torch.float32, device="cuda")
    Y = torch.zeros_like(X)
    fn = lib.sg_ffn_forward_batch_dense if args.dense else lib.sg_ffn_forward_batch
    for _ in range(3):
        check(fn(ctx.handle, layer.handle, C.c_void_p(X.data_ptr()), B, C.c_void_p(Y.data_ptr()), None))
    torch.cuda.synchronize()
    check(lib.sg_ctx_enable_tc_trace(ctx.handle, 8192))
    check(fn(ctx.handle, layer.handle, C.c_void_p(X.data_ptr()), B, C.c_void_p(Y.data_ptr()), None))
    out = np.zeros((8192, 8), dtype=np.uint64)
    n = C.c_int32(0)
    check(lib.sg_ctx_read_tc_trace(ctx.handle, None, 8192, out.ctypes.data_as(C.c_void_p), C.byref(n)))
    tr = out[:n.value].astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    rel = (tr[:, :5] - t0) / 1e3
    mid = np.where(tr[:, 6:8] > 0, (tr[:, 6:8] - t0) / 1e3, np.nan)
    codes = np.zeros(n.value, dtype=np.int32)
    check(lib.sg_tc_unit_codes(ctx.handle, codes.ctypes.data_as(C.c_void_p), n.value))
    order = codes >> 24
    end = rel[:, 4].max()
    print(f"{'dense' if args.dense else 'sparse'} B={B}: {n.value} units, launch span {end:.1f} us")
    print(f"{'type':6s} {'n':>5s} {'claim0':>8s} {'claim1':>8s} {'done0':>8s} {'done1':>8s} "
          f"{'wait':>7s} {'load':>7s} {'mma':>7s} {'epi':>7s} {'e.part':>7s} {'e.arr':>7s} {'e.fin':>7s}")
    for t, name in TYPES.items():
        sel = order == t
        if not sel.any():
            continue
        r = rel[sel]
        wait = r[:, 1] - r[:, 0]
        load = r[:, 2] - r[:, 1]
        mma = r[:, 3] - r[:, 2]
        epi = r[:, 4] - r[:, 3]
        mm = mid[sel]
        ep = np.nanmean(mm[:, 0] - r[:, 3]) if np.isfinite(mm[:, 0]).any() else float("nan")
        ea = np.nanmean(mm[:, 1] - mm[:, 0]) if np.isfinite(mm[:, 1]).any() else float("nan")
        ef = np.nanmean(r[:, 4] - mm[:, 1]) if np.isfinite(mm[:, 1]).any() else float("nan")
        if t == 1:  # X: no loads, no MMA
            load = mma = np.full_like(load, np.nan)
        print(f"{name:6s} {sel.sum():5d} {r[:, 0].min():8.1f} {r[:, 0].max():8.1f} {r[:, 4].min():8.1f} "
              f"{r[:, 4].max():8.1f} {wait.mean():7.2f} {np.nanmean(load):7.2f} {np.nanmean(mma):7.2f} "
              f"{epi.mean():7.2f} {ep:7.2f} {ea:7.2f} {ef:7.2f}")
    if args.fin:
        sel = order == 4
        r = tr[sel]
        ready, first, ewait = (r[:, 1] - t0) / 1e3, (r[:, 6] - t0) / 1e3, r[:, 2] / 1e3
        done = (r[:, 3] - t0) / 1e3
        print(f"DOWN (fintrace): ready {ready.mean():.1f} first stage {first.mean():.1f} "
              f"(+{(first - ready).mean():.2f}) accumulator done {done.mean():.1f} "
              f"(first stage -> done {(done - first).mean():.2f} us, of which waiting for free stages "
              f"{ewait.mean():.2f})")
        nstg, nf, fns = r[:, 5] >> 40, (r[:, 5] >> 32) & 0xff, (r[:, 5] & 0xffffffff) / 1e3
        print(f"  stages per unit {nstg.mean():.1f} (max {nstg.max()}), block-flag refetches {nf.mean():.1f}, "
              f"time in them {fns.mean():.2f} us; in the block walker {r[:, 7].mean() / 1e3:.2f} us")
        return
    sms = tr[:, 5]
    busy = np.zeros(int(sms.max()) + 1)
    for k in range(n.value):
        busy[sms[k]] += rel[k, 4] - rel[k, 1]
    print(f"SM busy (inputs ready -> epilogue end) mean {busy.mean():.1f} us of {end:.1f}")
    for sm in sorted(set(sms.tolist()))[:args.sms]:
        ks = np.nonzero(sms == sm)[0]
        ks = ks[np.argsort(rel[ks, 0])]
        print(f"SM {sm}: " + " | ".join(
            f"{TYPES.get(int(order[k]), '?')}({(codes[k] >> 8) & 0xffff},{codes[k] & 0xff}) c{rel[k, 0]:.1f} r{rel[k, 1]:.1f} "
            f"l{rel[k, 2]:.1f} e{rel[k, 3]:.1f}-{rel[k, 4]:.1f}" for k in ks))


if __name__ == "__main__":
    main()
