#!/usr/bin/env python
"""Small inputs through every device path of the library, for compute-sanitizer
(memcheck / synccheck / racecheck, one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py

single-token executor (all pipelines), predict_mask, a chained stack launch (chain 0 /
1 / 2, with stack sets), the tensor-core batch kernel (sparse B = 3 and 17, dense
comparator), the offline producer and exact f64 mask. Exits 0 when every call
returned SG_OK (the sanitizer decides the rest)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2603_14110_b200 import DeviceLayer, Pipeline
    from paper_2603_14110_b200 import _capi as capi
    from paper_2603_14110_b200.ffn_exec import Context, check
    from paper_2603_14110_b200.offline import build_predictor, damage_weights, greedy_calibrate, proxy_scores
    from paper_2603_14110_b200.synthetic import SyntheticConfig, make_synthetic_fixture

    lib = capi.lib()
    d, D, r = 256, 1024, 32
    fx = make_synthetic_fixture(SyntheticConfig(hidden=d, inter=D, calib_tokens=256, eval_tokens=24, seed=4))
    pred = build_predictor(fx.weights.gate, fx.calib, r).predictor
    pred.bias = greedy_calibrate(proxy_scores(pred, fx.calib), damage_weights(fx.weights, fx.calib), 8, 0.5).bias
    layer = DeviceLayer(fx.weights, pred, device=0)
    x = fx.eval[:, 0]
    for p in (Pipeline.Dense, Pipeline.Parallel, Pipeline.Sequential):
        layer.forward(x, p)
    layer.predict_mask(x)
    # stack of 3 layers, every chain mode, with the per-layer sets recorded
    ctx = Context(0, d, D, r)
    layers = (C.c_void_p * 3)(*[layer.handle] * 3)
    xs = torch.tensor(np.ascontiguousarray(fx.eval[:, :3].T), dtype=torch.float32, device="cuda")
    ys = torch.zeros_like(xs)
    check(lib.sg_ctx_enable_stack_sets(ctx.handle, 1))
    for chain in (0, 1, 2):
        check(lib.sg_ffn_forward_layers(ctx.handle, layers, 3, int(Pipeline.Sequential), C.c_void_p(xs.data_ptr()),
                                        C.c_void_p(ys.data_ptr()), chain, None))
    torch.cuda.synchronize()
    # tensor-core batch kernel: sparse (odd and > 16 tokens) and the dense comparator
    for B in (3, 17):
        layer.forward_batch(np.ascontiguousarray(fx.eval[:, :B].T))
    layer.forward_batch_dense(np.ascontiguousarray(fx.eval[:, :8].T))
    # offline producer + exact mask
    A = np.ascontiguousarray(pred.A, dtype=np.float64)
    Bm = np.ascontiguousarray(pred.B, dtype=np.float64)
    bias = np.ascontiguousarray(pred.bias, dtype=np.float64)
    mask = np.zeros(D, dtype=np.uint8)
    cnt = C.c_int64(0)
    xd = np.ascontiguousarray(x, dtype=np.float64)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    check(lib.sg_predict_mask_f64(0, p(A), p(Bm), p(bias), D, r, d, p(xd), p(mask), C.byref(cnt)))
    torch.cuda.synchronize()
    print("sanitize_case: all calls ok")


if __name__ == "__main__":
    main()
