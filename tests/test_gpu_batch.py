"""GPU parity of batched decode (sg_ffn_forward_batch, BASELINE.json configs[4]).

B >= 2 runs the tensor-core kernel (csrc/sg_batch_tc.cu: tcgen05.mma, TMEM
accumulators, TMA tile::gather4 of the union rows); B = 1 the persistent
single-token executor.

Every token of a batch must get its own single-token result: its predicted and
survivor sets (bit-exact up to the near-threshold band) and y (Y_RTOL), against
the f64 oracle run on that token alone (tests/parity_util.py rules), and the
reference's ExecStats formulas on its own counts.
"""
import numpy as np
import pytest

from paper_2603_14110_b200 import DataError, DeviceLayer, Pipeline
from paper_2603_14110_b200.model import CONFIGS, build_host_layer, upload
from parity_util import Y_RTOL, check_token, quantize_layer
from test_gpu_parity import _calibrated_layer
from test_gpu_scale import _host_q

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B", [1, 3, 4, 5, 7, 8, 12, 16, 17, 64])
def test_batch_tokens_match_single_token_oracle(B):
    d, D, r = 512, 2048, 64
    fx, pred = _calibrated_layer(d, D, r, seed=9, calib=1024)
    q = quantize_layer(fx.weights.gate, fx.weights.up, fx.weights.down, pred.A, pred.B, pred.bias)
    layer = DeviceLayer(fx.weights, pred)
    rng = np.random.default_rng(B)
    X = fx.eval[:, rng.integers(0, fx.eval.shape[1], B)].T + 0.1 * rng.standard_normal((B, d))
    Y, stats, P, V = layer.forward_batch(X)
    worst = 0.0
    for b in range(B):
        diag = check_token(q, X[b], Y[b], P[b], V[b])
        worst = max(worst, diag["rel"])
        st = stats[b]
        assert (st.predicted_active, st.revalidated) == (len(P[b]), len(V[b]))
        assert st.multiplies == r * (d + D) + d * len(P[b]) + 2 * d * len(V[b])
        assert st.pipeline == Pipeline.Sequential
    assert worst <= Y_RTOL
    # deterministic, and token b's result does not depend on its batch mates
    Y2, _, P2, _ = layer.forward_batch(X)
    assert np.array_equal(Y, Y2)
    if B > 1:
        Y1, _, P1, _ = layer.forward_batch(X[:1])
        assert [p.tolist() for p in P1] == [P[0].tolist()]


def test_batch_full_size_7b():
    cfg = CONFIGS["7b"]
    d, D = cfg["d"], cfg["D"]
    h = build_host_layer(d, D, 0, seed=2, rank=256, sparsity=0.5, eval_tokens=16)
    layer = upload(h, d, D, 0, 256)
    q = _host_q(h)
    Y, stats, P, V = layer.forward_batch(h.xs.T)
    for b in range(16):
        diag = check_token(q, h.xs[:, b], Y[b], P[b], V[b])
        assert diag["rel"] <= Y_RTOL


def test_batch_rejects_bad_input():
    fx, pred = _calibrated_layer(64, 256, 8, seed=3)
    layer = DeviceLayer(fx.weights, pred)
    with pytest.raises(Exception):
        layer.forward_batch(np.ones((65, 64)))
    bad = np.ones((2, 64))
    bad[1, 3] = np.nan
    with pytest.raises(DataError):
        layer.forward_batch(bad)


@pytest.mark.parametrize("d,D,r,act", [(500, 1000, 64, 0), (512, 1408, 256, 1), (1024, 3000, 128, 0)])
def test_batch_ragged_shapes_and_drelu(d, D, r, act):
    """hidden not a multiple of 64, inter not a multiple of the 256-neuron block,
    rank 64 / 128 / 256 (one or two M = 128 predictor sub-tiles), dReLU."""
    from paper_2603_14110_b200 import Activation
    fx, pred = _calibrated_layer(d, D, r, seed=21 + d, calib=1024, act=Activation(act))
    q = quantize_layer(fx.weights.gate, fx.weights.up, fx.weights.down, pred.A, pred.B, pred.bias)
    layer = DeviceLayer(fx.weights, pred)
    rng = np.random.default_rng(d)
    for B in (2, 9, 33, 47):  # (47: past 42 tokens the sparse GU unit takes 3N TMEM columns)
        X = fx.eval[:, rng.integers(0, fx.eval.shape[1], B)].T + 0.1 * rng.standard_normal((B, d))
        Y, stats, P, V = layer.forward_batch(X)
        for b in range(B):
            diag = check_token(q, X[b], Y[b], P[b], V[b], act=act)
            assert diag["rel"] <= Y_RTOL


@pytest.mark.parametrize("B", [2, 8, 16, 40, 64])
def test_dense_batch_matches_single_token_dense(B):
    """sg_ffn_forward_batch_dense (every row on the tensor cores) against the dense
    executor per token (ffn_exec.hpp:103-122), and against the f64 dense oracle."""
    import oracle as O
    d, D, r = 512, 2048, 64
    fx, pred = _calibrated_layer(d, D, r, seed=4, calib=1024)
    q = quantize_layer(fx.weights.gate, fx.weights.up, fx.weights.down, pred.A, pred.B, pred.bias)
    layer = DeviceLayer(fx.weights, pred)
    rng = np.random.default_rng(B)
    X = fx.eval[:, rng.integers(0, fx.eval.shape[1], B)].T + 0.1 * rng.standard_normal((B, d))
    X = X.astype(np.float32).astype(np.float64)
    Y = layer.forward_batch_dense(X)
    for b in range(B):
        ref, _ = O.dense_ffn(q["gate"], q["up"], q["down"], X[b])
        assert np.linalg.norm(Y[b] - ref) <= Y_RTOL * np.linalg.norm(ref)
        one = layer.forward(X[b], Pipeline.Dense).y
        assert np.linalg.norm(Y[b] - one) <= Y_RTOL * np.linalg.norm(one)


def test_batch_device_entry_flags_nonfinite():
    """The device entry has no host check: the kernel flags a non-finite token and
    sg_ctx_read_batch raises DataError (ffn_exec.hpp:61-63)."""
    import ctypes as C

    import torch

    from paper_2603_14110_b200 import _capi as capi
    from paper_2603_14110_b200.ffn_exec import check
    fx, pred = _calibrated_layer(256, 768, 32, seed=6)
    layer = DeviceLayer(fx.weights, pred)
    ctx = layer.context()
    for B in (1, 5, 20):
        X = torch.tensor(np.tile(fx.eval[:, :1].T, (B, 1)), dtype=torch.float32, device="cuda")
        X[B - 1, 7] = float("inf")
        Y = torch.zeros_like(X)
        sh = torch.cuda.current_stream().cuda_stream
        check(capi.lib().sg_ffn_forward_batch(ctx.handle, layer.handle, C.c_void_p(X.data_ptr()), B,
                                              C.c_void_p(Y.data_ptr()), C.c_void_p(sh)))
        with pytest.raises(DataError):
            check(capi.lib().sg_ctx_read_batch(ctx.handle, C.c_void_p(sh), B, None, None, None))


@pytest.mark.parametrize("dense,B", [(0, 12), (1, 12), (0, 1)])
def test_batch_residual_input_equals_summed_input(dense, B):
    """sg_ffn_forward_batch_res (x_b = h_b + r_b formed inside the launch, the residual
    chain of the batched bench) gives exactly the result of the same call on the
    fp32 sums."""
    import ctypes as C

    import torch

    from paper_2603_14110_b200 import _capi as capi
    from paper_2603_14110_b200.ffn_exec import Context, check

    d, D, r = 512, 2048, 64
    fx, pred = _calibrated_layer(d, D, r, seed=5, calib=1024)
    layer = DeviceLayer(fx.weights, pred)
    rng = np.random.default_rng(3)
    H = torch.tensor(fx.eval[:, rng.integers(0, fx.eval.shape[1], B)].T.copy(), dtype=torch.float32, device="cuda")
    R = torch.tensor(0.1 * rng.standard_normal((B, d)), dtype=torch.float32, device="cuda")
    S = (H + R).contiguous()
    ctx = Context(0, d, D, r)
    lib = capi.lib()
    Y1, Y2 = torch.zeros_like(H), torch.zeros_like(H)
    check(lib.sg_ffn_forward_batch_res(ctx.handle, layer.handle, C.c_void_p(H.data_ptr()),
                                       C.c_void_p(R.data_ptr()), B, C.c_void_p(Y1.data_ptr()), dense,
                                       None, None, None))
    check(lib.sg_ffn_forward_batch_res(ctx.handle, layer.handle, C.c_void_p(S.data_ptr()), None, B,
                                       C.c_void_p(Y2.data_ptr()), dense, None, None, None))
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    assert float(Y1.abs().sum()) > 0


@pytest.mark.parametrize("chain", [1, 2])
def test_batch_prepared_next_input_equals_plain_chain(chain):
    """A chain of batched calls where each launch's y finishers also write the next
    call's X^T (`next` / `next_xs`) gives exactly the results of the same chain run
    without that, call by call (the next call then runs no x split)."""
    import ctypes as C

    import torch

    from paper_2603_14110_b200 import _capi as capi
    from paper_2603_14110_b200.ffn_exec import Context, check

    d, D, r, B, L = 512, 2048, 64, 9, 3
    layers = []
    for l in range(L):
        fx, pred = _calibrated_layer(d, D, r, seed=30 + l, calib=1024)
        layers.append(DeviceLayer(fx.weights, pred))
    rng = np.random.default_rng(7)
    H = [torch.tensor(0.5 * rng.standard_normal((B, d)), dtype=torch.float32, device="cuda") for _ in range(L)]
    lib = capi.lib()

    def run(prep):
        ctx = Context(0, d, D, r)
        Y = [torch.zeros_like(H[0]) for _ in range(L)]
        for l in range(L):
            if l == 0:
                x, res = H[0], None
            elif chain == 1:
                x, res = Y[l - 1], None
            else:
                x, res = H[l], Y[l - 1]
            nxt = layers[l + 1].handle if prep and l + 1 < L else None
            nxs = C.c_void_p(H[l + 1].data_ptr()) if prep and l + 1 < L and chain == 2 else None
            check(lib.sg_ffn_forward_batch_res(ctx.handle, layers[l].handle, C.c_void_p(x.data_ptr()),
                                               C.c_void_p(res.data_ptr()) if res is not None else None, B,
                                               C.c_void_p(Y[l].data_ptr()), 0, nxt, nxs, None))
        torch.cuda.synchronize()
        return Y

    Ya, Yb = run(False), run(True)
    for l in range(L):
        assert torch.equal(Ya[l], Yb[l]), l


@pytest.mark.parametrize("tile_u", [2000, 300])
def test_batch_gathered_down_rows(tile_u, monkeypatch):
    """The down stage's row-gather path (survivor rows of a block gathered by cp.async
    instead of the block tiled; the default tiles every block with a survivor):
    SG_TC_TILE_U above 1024 gathers every block, 300 mixes gathered and tiled blocks
    inside one range (runs broken by gathered blocks)."""
    monkeypatch.setenv("SG_TC_TILE_U", str(tile_u))
    d, D, r = 512, 2048, 64
    fx, pred = _calibrated_layer(d, D, r, seed=11, calib=1024)
    q = quantize_layer(fx.weights.gate, fx.weights.up, fx.weights.down, pred.A, pred.B, pred.bias)
    layer = DeviceLayer(fx.weights, pred)
    rng = np.random.default_rng(tile_u)
    for B in (3, 16, 40):
        X = fx.eval[:, rng.integers(0, fx.eval.shape[1], B)].T + 0.1 * rng.standard_normal((B, d))
        Y, stats, P, V = layer.forward_batch(X)
        for b in range(B):
            diag = check_token(q, X[b], Y[b], P[b], V[b])
            assert diag["rel"] <= Y_RTOL


def test_forward_batch_residual_python_api():
    """DeviceLayer.forward_batch_residual (Python mirror of sg_ffn_forward_batch_res)
    equals forward_batch on the fp32 sums, stats included."""
    import torch
    d, D, r, B = 512, 2048, 64, 6
    fx, pred = _calibrated_layer(d, D, r, seed=6, calib=1024)
    layer = DeviceLayer(fx.weights, pred)
    rng = np.random.default_rng(9)
    H = torch.tensor(fx.eval[:, :B].T.copy(), dtype=torch.float32, device="cuda")
    R = torch.tensor(0.1 * rng.standard_normal((B, d)), dtype=torch.float32, device="cuda")
    Y, st = layer.forward_batch_residual(H, R)
    Y2, st2, _, _ = layer.forward_batch((H + R).cpu().numpy())
    assert np.array_equal(Y.double().cpu().numpy(), Y2)
    assert [(s.predicted_active, s.revalidated) for s in st] == [(s.predicted_active, s.revalidated) for s in st2]
