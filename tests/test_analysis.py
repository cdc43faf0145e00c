"""Caller-side metrics (paper_2603_14110_b200/analysis.py) against the cases of
/root/reference/proj/tests/analysis_tests.cpp:227-322. roc_auc is host-only (CPU);
layer_metrics drives the GPU executor (gpu marker)."""
import numpy as np
import pytest

from paper_2603_14110_b200 import DataError, FfnWeights, Predictor
from paper_2603_14110_b200.analysis import (fnv1a64, format_stream, hex64, layer_metrics,
                                            roc_auc, run_record, run_stream)


def brute_force_auc(scores, labels):
    pos = [s for s, l in zip(scores, labels) if l]
    neg = [s for s, l in zip(scores, labels) if not l]
    acc = 0.0
    for p in pos:
        for n in neg:
            acc += 1.0 if p > n else (0.5 if p == n else 0.0)
    return acc / (len(pos) * len(neg))


def test_roc_auc_basics():  # analysis_tests.cpp:227-241
    assert roc_auc([1, 2, 3, 4], [0, 0, 1, 1]) == 1.0
    assert roc_auc([5, 5, 5, 5], [0, 1, 0, 1]) == 0.5
    assert roc_auc([1, 2, 3, 4], [0, 1, 0, 1]) == 0.75
    with pytest.raises(DataError):
        roc_auc([1, 2], [1, 1])
    with pytest.raises(DataError):
        roc_auc([1, 2], [0, 0])


def test_roc_auc_equals_brute_force():  # :243-268 (ties forced by a small alphabet)
    rng = np.random.default_rng(23)
    for _ in range(100):
        n = int(rng.integers(2, 201))
        scores = rng.integers(0, 10, n) / 3.0
        labels = rng.random(n) < 0.5
        labels[0] = True
        labels[1] = False
        assert roc_auc(scores, labels) == brute_force_auc(scores, labels)


def _ffn(rng, d, D):
    return FfnWeights(rng.standard_normal((D, d)), rng.standard_normal((D, d)), rng.standard_normal((d, D)))


@pytest.mark.gpu
def test_layer_metrics_controlled_predictors():  # :270-322
    rng = np.random.default_rng(31)
    w = _ffn(rng, 8, 24)
    X = rng.standard_normal((8, 16))
    exact = Predictor(w.gate.copy(), np.eye(8), np.zeros(24), 8)
    row = layer_metrics(w, exact, X, 3)
    assert row.layer == 3 and row.recall == 1.0 and row.roc_auc == 1.0
    assert row.mean_rel_output_error <= 1e-5  # bf16 weights on the GPU (reference: f64, 1e-12)
    assert row.predicted_sparsity == row.realized_sparsity
    off = Predictor(w.gate.copy(), np.eye(8), np.full(24, -1e12), 8)
    row = layer_metrics(w, off, X)
    assert row.recall == 0.0 and row.predicted_sparsity == 1.0
    pred = Predictor(w.gate.copy(), np.eye(8), rng.standard_normal(24), 8)
    row = layer_metrics(w, pred, X)
    g = w.gate @ X
    pre = pred.A @ (pred.B @ X) + pred.bias[:, None]
    rec = [((pre[:, t] > 0) & (g[:, t] > 0)).sum() / (g[:, t] > 0).sum()
           for t in range(16) if (g[:, t] > 0).any()]
    assert abs(row.recall - np.mean(rec)) <= 1e-12
    assert abs(row.roc_auc - brute_force_auc(pre.T.reshape(-1), (g > 0).T.reshape(-1))) <= 1e-12


def test_fnv1a64_and_hex64():
    """sparsegate_main.cpp:73-87. The reference's offset basis literal is
    1469598103934665603 (the published FNV-1a basis is 14695981039346656037): the
    stream must hash like the reference, so the restatement keeps its constant."""
    basis, prime = 1469598103934665603, 1099511628211
    assert fnv1a64(b"") == basis
    assert fnv1a64(b"a") == ((basis ^ 0x61) * prime) % 2 ** 64 == 0x44BD8AD473CD9906
    h = basis
    for b in b"foobar":
        h = ((h ^ b) * prime) % 2 ** 64
    assert fnv1a64(b"foobar") == h
    assert hex64(1) == "0000000000000001" and hex64(fnv1a64(b"a")) == "44bd8ad473cd9906"


def test_run_stream_format():
    """cmd_run records (sparsegate_main.cpp:251-258): compact, keys in std::map order."""
    class St:
        predicted_sparsity, realized_sparsity, multiplies = 0.5, 0.75, 12

    class R:
        y, stats = np.array([1.0, 0.0]), St()

    rec = run_record(3, R())
    h = hex64(fnv1a64(np.array([1.0, 0.0], dtype="<f8").tobytes()))
    assert format_stream([rec]) == ('{"multiplies":12,"output_hash":"%s","predicted_sparsity":0.5,'
                                    '"realized_sparsity":0.75,"token_index":3}\n' % h)


@pytest.mark.gpu
def test_run_stream_gpu():
    """The stream from GPU runs: byte-identical reruns, the reference's stats fields
    (multiplies exact unless a near-threshold neuron flips), dense multiplies 3dD."""
    import json
    import oracle as O
    from parity_util import q_f32, quantize_layer
    from test_gpu_parity import _calibrated_layer
    d, D, r = 256, 1024, 32
    fx, pred = _calibrated_layer(d, D, r, seed=5)
    X = fx.eval[:, :6]
    s1 = run_stream(fx.weights, pred, X)
    assert s1 == run_stream(fx.weights, pred, X)
    q = quantize_layer(fx.weights.gate, fx.weights.up, fx.weights.down, pred.A, pred.B, pred.bias)
    for t, line in enumerate(s1.splitlines()):
        rec = json.loads(line)
        assert rec["token_index"] == t and list(rec) == sorted(rec)
        o = O.sparse_ffn(q["gate"], q["up"], q["down"], q["A"], q["B"], q["bias"], q_f32(X[:, t]))
        assert abs(rec["multiplies"] - o.stats.multiplies) <= 4 * d
    for line in run_stream(fx.weights, pred, X, mode="dense").splitlines():
        assert json.loads(line)["multiplies"] == 3 * d * D
    with pytest.raises(DataError):
        run_stream(fx.weights, pred, X, mode="bogus")
