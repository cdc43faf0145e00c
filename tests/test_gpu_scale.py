"""GPU parity at BASELINE.json sizes, for d_ff shards, and for multi-layer launches.

* Full-size layers of configs[1..3] (7B ReGLU, Mistral-7B dReLU, 13B ReGLU),
  built exactly as the bench builds them (paper_2603_14110_b200.model), checked
  token by token against the f64 oracle under the rules of tests/parity_util.py.
* d_ff sharding on one GPU: the shards of a layer, run one after
  the other, must sum to the unsharded layer and their index sets must be the
  global sets (the exchange itself is covered on CPU by tests/test_sharded_cpu.py).
* The multi-layer persistent launch (sg_ffn_forward_layers) must equal layer-by-
  layer launches bit for bit, with and without chaining.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2603_14110_b200 import (Activation, DeviceLayer, Pipeline, bf16_to_f64, read_sets,
                                   read_stats)
from paper_2603_14110_b200 import _capi as capi
from paper_2603_14110_b200.ffn_exec import Context, check
from paper_2603_14110_b200.model import CONFIGS, build_host_layer, upload
from paper_2603_14110_b200.sharded import shard_indices, stats_from_counts
from parity_util import Y_RTOL, check_token, q_f32, quantize_layer
from test_gpu_parity import _calibrated_layer

pytestmark = pytest.mark.gpu


def _host_q(h):
    return dict(gate=bf16_to_f64(h.gate), up=bf16_to_f64(h.up),
                down=np.ascontiguousarray(bf16_to_f64(h.down_t).T), A=bf16_to_f64(h.A),
                B=bf16_to_f64(h.B), bias=q_f32(h.bias))


@pytest.mark.parametrize("config", ["7b", "mistral", "13b"])
def test_full_size_layer_parity(config):
    cfg = CONFIGS[config]
    d, D, act = cfg["d"], cfg["D"], cfg["act"]
    h = build_host_layer(d, D, act, seed=1, rank=256, sparsity=0.5, eval_tokens=3)
    layer = upload(h, d, D, act, 256)
    q = _host_q(h)
    ctx = layer.context()
    for t in range(h.xs.shape[1]):
        x = h.xs[:, t]
        res = layer.forward(x, Pipeline.Sequential, ctx)
        P, V, _, _ = read_sets(ctx, D)
        diag = check_token(q, x, res.y, P, V, act=act)
        assert diag["rel"] <= Y_RTOL
        # the calibrated operating point of the bench: p ~ D/2, v ~ 0.1 D
        assert 0.3 * D < diag["p"] < 0.7 * D and 0.03 * D < diag["v"] < 0.2 * D
        st = res.stats
        assert st.multiplies == 256 * (d + D) + d * len(P) + 2 * d * len(V)


@pytest.mark.parametrize("shards,interleave", [(2, False), (3, False), (2, True), (3, True)])
def test_shards_sum_to_the_full_layer(shards, interleave):
    d, D, r = 512, 1500, 64
    fx, pred = _calibrated_layer(d, D, r, seed=77, calib=1024)
    q = quantize_layer(fx.weights.gate, fx.weights.up, fx.weights.down, pred.A, pred.B, pred.bias)
    parts = [DeviceLayer(fx.weights, pred, shard_index=k, shard_count=shards,
                         shard_interleave=interleave) for k in range(shards)]
    for k, lay in enumerate(parts):
        idx = shard_indices(D, k, shards, interleave)
        assert lay.local_inter == len(idx)
        assert [lay.global_index(i) for i in (0, len(idx) - 1)] == [idx[0], idx[-1]]
    for t in range(4):
        x = fx.eval[:, t]
        y = np.zeros(d)
        P, V = [], []
        p = v = 0
        for lay in parts:
            ctx = lay.context()
            res = lay.forward(x, Pipeline.Sequential, ctx)
            y += res.y
            Pk, Vk, _, _ = read_sets(ctx, lay.local_inter)
            P += Pk.tolist()
            V += Vk.tolist()
            p += res.stats.predicted_active
            v += res.stats.revalidated
        P, V = sorted(P), sorted(V)
        diag = check_token(q, x, y, P, V)
        assert diag["rel"] <= Y_RTOL
        st = stats_from_counts(d, D, r, Pipeline.Sequential, p, v)
        assert st.multiplies == r * (d + D) + d * len(P) + 2 * d * len(V)
        if diag["dP"] == 0 and diag["dV"] == 0:
            o = diag["oracle"].stats
            assert (st.multiplies, st.predicted_sparsity, st.realized_sparsity) == \
                (o.multiplies, o.predicted_sparsity, o.realized_sparsity)


def _stack(layers, xs, chain, pipeline=Pipeline.Sequential):
    import torch
    d = layers[0].hidden
    ctx = Context(0, d, max(l.local_inter for l in layers), max(l.rank for l in layers))
    arr = (C.c_void_p * len(layers))(*[l.handle.value for l in layers])
    xt = torch.tensor(np.asarray(xs, dtype=np.float32), device="cuda")
    yt = torch.zeros_like(xt)
    sh = torch.cuda.current_stream().cuda_stream
    check(capi.lib().sg_ffn_forward_layers(ctx.handle, arr, len(layers), int(pipeline),
                                           C.c_void_p(xt.data_ptr()), C.c_void_p(yt.data_ptr()),
                                           int(chain), C.c_void_p(sh)))
    st = (capi.sg_exec_stats * len(layers))()
    check(capi.lib().sg_ctx_read_stack_stats(ctx.handle, C.c_void_p(sh), len(layers), st))
    return yt.double().cpu().numpy(), [(s.predicted_active, s.revalidated) for s in st]


@pytest.mark.parametrize("pipeline,hot", [(Pipeline.Sequential, 0), (Pipeline.Sequential, 5),
                                          (Pipeline.Parallel, 0), (Pipeline.Dense, 0)])
def test_stack_launch_equals_layer_launches(pipeline, hot):
    """hot > 0: the next layer's hot prefix is fetched during the previous layer's
    tail in a stack, at layer start otherwise; the results must not differ."""
    import torch
    d, D, r = 512, 1408, 64
    layers, xs = [], []
    for s in range(3):
        fx, pred = _calibrated_layer(d, D, r, seed=100 + s)
        layers.append(DeviceLayer(fx.weights, pred))
        layers[-1].set_hot_rows(hot)
        xs.append(fx.eval[:, 0])
    xs = np.stack(xs).astype(np.float32).astype(np.float64)
    ys, stats = _stack(layers, xs, chain=0, pipeline=pipeline)
    for l, lay in enumerate(layers):
        ctx = lay.context()
        res = lay.forward(xs[l], pipeline, ctx)
        assert np.array_equal(ys[l], res.y), f"layer {l}"
        if pipeline != Pipeline.Dense:
            assert stats[l] == (res.stats.predicted_active, res.stats.revalidated)
    # chained: layer l+1 reads layer l's output (fp32 on device)
    yc, _ = _stack(layers, xs, chain=1, pipeline=pipeline)
    x = xs[0]
    for l, lay in enumerate(layers):
        res = lay.forward(x, pipeline)
        assert np.array_equal(yc[l], res.y), f"chained layer {l}"
        x = res.y.astype(np.float32).astype(np.float64)
    torch.cuda.synchronize()


def test_repeated_stacks_on_one_context():
    """Layers inside a stack exchange t and y as tagged values instead of grid
    barriers; the tags derive from the context's barrier counters. Stacks of
    different depths, single-layer calls and predictor-only calls interleaved on
    ONE context must keep giving the same bits (a stale tag would let a reader
    take a previous launch's value)."""
    import torch
    d, D, r = 512, 1408, 64
    layers, xs = [], []
    for s in range(4):
        fx, pred = _calibrated_layer(d, D, r, seed=200 + s)
        layers.append(DeviceLayer(fx.weights, pred))
        xs.append(fx.eval[:, 0])
    xt = torch.tensor(np.asarray(xs, dtype=np.float32), device="cuda")
    ctx = Context(0, d, D, r)
    sh = torch.cuda.current_stream().cuda_stream

    def stack(n, chain):
        arr = (C.c_void_p * n)(*[l.handle.value for l in layers[:n]])
        yt = torch.zeros_like(xt)
        check(capi.lib().sg_ffn_forward_layers(ctx.handle, arr, n, int(Pipeline.Sequential),
                                               C.c_void_p(xt.data_ptr()), C.c_void_p(yt.data_ptr()),
                                               int(chain), C.c_void_p(sh)))
        return yt[:n].double().cpu().numpy()

    ref = {(n, c): stack(n, c) for n in (2, 4) for c in (0, 1)}
    for it in range(6):
        for n, c in ((4, 1), (2, 0), (4, 0), (2, 1)):
            assert np.array_equal(stack(n, c), ref[(n, c)]), (it, n, c)
        layers[it % 4].forward(xs[it % 4], Pipeline.Sequential, ctx)
        layers[it % 4].predict_mask(xs[it % 4], ctx)
    torch.cuda.synchronize()


@pytest.mark.parametrize("shards", [1, 2])
def test_layout_order_keeps_parity(shards):
    """A neuron layout order (sg_layer_desc.neuron_order) moves work between CTAs
    only: sets (reported in global indices, ascending) and y stay within parity."""
    from paper_2603_14110_b200 import round_bf16
    d, D, r = 512, 1500, 64
    fx, pred = _calibrated_layer(d, D, r, seed=31, calib=1024)
    q = quantize_layer(fx.weights.gate, fx.weights.up, fx.weights.down, pred.A, pred.B, pred.bias)
    order = np.random.default_rng(3).permutation(D)
    raw = dict(hidden=d, inter=D, rank=r, activation=0, gate=round_bf16(fx.weights.gate),
               up=round_bf16(fx.weights.up), down_t=round_bf16(np.ascontiguousarray(fx.weights.down.T)),
               A=round_bf16(pred.A), B=round_bf16(pred.B), bias=pred.bias.astype(np.float32),
               order=order)
    parts = [DeviceLayer(raw=raw, shard_index=k, shard_count=shards) for k in range(shards)]
    for k, lay in enumerate(parts):
        mine = set(shard_indices(D, k, shards).tolist())
        gl = [lay.global_index(i) for i in range(lay.local_inter)]
        assert set(gl) == mine
        pos = {g: i for i, g in enumerate(order)}
        assert [pos[g] for g in gl] == sorted(pos[g] for g in gl)  # layout follows the order
    for t in range(4):
        x = fx.eval[:, t]
        y = np.zeros(d)
        P, V = [], []
        for lay in parts:
            ctx = lay.context()
            y += lay.forward(x, Pipeline.Sequential, ctx).y
            Pk, Vk, _, _ = read_sets(ctx, lay.local_inter)
            assert list(Pk) == sorted(Pk) and list(Vk) == sorted(Vk)
            P += Pk.tolist()
            V += Vk.tolist()
        diag = check_token(q, x, y, sorted(P), sorted(V))
        assert diag["rel"] <= Y_RTOL
    with pytest.raises(Exception):
        bad = dict(raw, order=np.zeros(D, dtype=np.int64))
        DeviceLayer(raw=bad)


@pytest.mark.parametrize("hot", [1, 7, 64])
def test_hot_prefix_keeps_parity(hot):
    """sg_layer_set_hot_rows on a layout whose block prefixes are NOT the hot
    neurons (ascending order): many prefetched rows are rejected by the mask and
    must be dropped. The item order stays ascending (the prefix is the block's
    first neurons), so the result is bit-identical to the hot-off run."""
    d, D, r = 512, 1500, 64
    fx, pred = _calibrated_layer(d, D, r, seed=41, calib=1024)
    q = quantize_layer(fx.weights.gate, fx.weights.up, fx.weights.down, pred.A, pred.B, pred.bias)
    base = DeviceLayer(fx.weights, pred)
    hl = DeviceLayer(fx.weights, pred)
    hl.set_hot_rows(hot)
    for t in range(6):
        x = fx.eval[:, t]
        ctx = base.context()
        r0 = base.forward(x, Pipeline.Sequential, ctx)
        P0, V0, g0, z0 = read_sets(ctx, D)
        r1 = hl.forward(x, Pipeline.Sequential, ctx)
        P1, V1, g1, z1 = read_sets(ctx, D)
        assert np.array_equal(P0, P1) and np.array_equal(V0, V1)
        assert np.array_equal(g0, g1) and np.array_equal(z0, z1)
        assert r0.stats == r1.stats
        diag = check_token(q, x, r1.y, P1, V1)
        assert diag["rel"] <= Y_RTOL
        assert np.array_equal(r0.y, r1.y)


@pytest.mark.parametrize("shards", [2, 3])
def test_bench_shards_with_layout_and_hot_prefix(shards):
    """Shards uploaded as the N > 1 bench does (model.upload: balanced hot-first layout
    per shard + 16-row hot prefix): their outputs sum to the oracle's y, their sets
    (global indices) partition the oracle's sets."""
    cfg = CONFIGS["tiny"]
    d, D = cfg["d"], cfg["D"]
    h = build_host_layer(d, D, 0, seed=6, rank=64, sparsity=0.5, eval_tokens=3)
    q = _host_q(h)
    parts = [upload(h, d, D, 0, 64, shard_index=k, shard_count=shards) for k in range(shards)]
    for t in range(h.xs.shape[1]):
        x = h.xs[:, t]
        y = np.zeros(d)
        P, V = [], []
        for lay in parts:
            ctx = lay.context()
            y += lay.forward(x, Pipeline.Sequential, ctx).y
            Pk, Vk, _, _ = read_sets(ctx, lay.local_inter)
            P += Pk.tolist()
            V += Vk.tolist()
        assert len(set(P)) == len(P) and len(set(V)) == len(V)
        diag = check_token(q, x, y, sorted(P), sorted(V))
        assert diag["rel"] <= Y_RTOL


def test_device_layer_container_round_trip(tmp_path):
    """save_device_layer / load_device_layer (tensor_io extension) reproduce the layer."""
    from paper_2603_14110_b200 import tensor_io as T
    cfg = CONFIGS["tiny"]
    d, D = cfg["d"], cfg["D"]
    h = build_host_layer(d, D, 0, seed=4, rank=64, sparsity=0.5, eval_tokens=2)
    a = upload(h, d, D, 0, 64, balance=False)
    T.save_device_layer(str(tmp_path), d, D, 0, h.gate, h.up, h.down_t, h.A, h.B, h.bias.astype(np.float32))
    b = T.load_device_layer(str(tmp_path))
    for t in range(2):
        ra, rb = a.forward(h.xs[:, t]), b.forward(h.xs[:, t])
        assert np.array_equal(ra.y, rb.y) and ra.stats == rb.stats
