"""GPU parity of batched decode (sg_ffn_forward_batch, BASELINE.json configs[4]).

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
    for b in (0, 7, 15):
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
