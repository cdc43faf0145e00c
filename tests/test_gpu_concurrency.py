"""Reentrancy: the reference executors are pure and are called concurrently from
worker threads (tools/sparsegate_main.cpp:241-259 runs them under
parallel_for, proj/include/sparsegate/parallel.hpp:26-50). The C ABI promises
the same for distinct sg_ctx objects sharing one sg_layer (include/sparsegate_c.h).

4 host threads x 4 contexts (one CUDA stream each) run the same layer at once
through the single-token, stack and batched entry points; every result must be
bit-identical to the same call made alone.
"""
import ctypes as C
import threading

import numpy as np
import pytest

from paper_2603_14110_b200 import DeviceLayer, Pipeline
from paper_2603_14110_b200 import _capi as capi
from paper_2603_14110_b200.ffn_exec import Context, check
from test_gpu_parity import _calibrated_layer

pytestmark = pytest.mark.gpu


def _batch(ctx, layer, xs, stream):
    B, d = xs.shape
    xh = np.ascontiguousarray(xs, dtype=np.float32)
    yh = np.zeros_like(xh)
    st = (capi.sg_exec_stats * B)()
    check(capi.lib().sg_ffn_forward_batch_host(ctx.handle, layer.handle,
                                               xh.ctypes.data_as(C.c_void_p), B,
                                               yh.ctypes.data_as(C.c_void_p), st, C.c_void_p(stream)))
    return yh, [(s.predicted_active, s.revalidated) for s in st]


def _stack(ctx, layers, xs, stream, chain):
    n, d = xs.shape
    arr = (C.c_void_p * n)(*[l.handle.value for l in layers])
    xh = np.ascontiguousarray(xs, dtype=np.float32)
    yh = np.zeros_like(xh)
    check(capi.lib().sg_ffn_forward_layers_host(ctx.handle, arr, n, int(Pipeline.Sequential),
                                                xh.ctypes.data_as(C.c_void_p),
                                                yh.ctypes.data_as(C.c_void_p), int(chain), None,
                                                C.c_void_p(stream)))
    return yh


def test_four_threads_four_contexts_one_layer():
    import torch
    d, D, r = 512, 2048, 64
    fx, pred = _calibrated_layer(d, D, r, seed=5)
    layer = DeviceLayer(fx.weights, pred)
    layer.set_hot_rows(4)
    stack_layers = [layer, layer, layer]
    xs = fx.eval[:, :8].T.astype(np.float32).astype(np.float64)

    def work(ctx, stream):
        out = {}
        for t in range(xs.shape[0]):
            for pipe in (Pipeline.Sequential, Pipeline.Parallel, Pipeline.Dense):
                r_ = layer.forward(xs[t], pipe, ctx, stream)
                out[("tok", t, int(pipe))] = (r_.y.copy(), r_.stats)
        out["stack0"] = _stack(ctx, stack_layers, xs[:3], stream, 0)
        out["stack1"] = _stack(ctx, stack_layers, xs[:3], stream, 1)
        for B in (3, 8):  # persistent-executor path and the batched path
            out[("batch", B)] = _batch(ctx, layer, xs[:B], stream)
        return out

    # the same calls, alone
    solo_ctx = Context(0, d, D, r)
    ref = work(solo_ctx, 0)

    ctxs = [Context(0, d, D, r) for _ in range(4)]
    streams = [torch.cuda.Stream() for _ in range(4)]
    results, errors = [None] * 4, []

    def run(i):
        try:
            res = None
            for _ in range(3):  # repeat so the threads genuinely overlap
                res = work(ctxs[i], streams[i].cuda_stream)
            results[i] = res
        except Exception as e:  # surfaced below
            errors.append(e)

    ths = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors
    for res in results:
        assert res.keys() == ref.keys()
        for k, v in ref.items():
            if isinstance(k, tuple) and k[0] == "tok":
                assert np.array_equal(res[k][0], v[0]), k
                assert res[k][1] == v[1], k
            elif isinstance(k, tuple) and k[0] == "batch":
                assert np.array_equal(res[k][0], v[0]), k
                assert res[k][1] == v[1], k
            else:
                assert np.array_equal(res[k], v), k
