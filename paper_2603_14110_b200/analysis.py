"""Caller-side predictor metrics over an evaluation batch,
restating /root/reference/proj/include/sparsegate/analysis.hpp:197-326 on top
of the GPU executor.

The executor calls (predict_mask, dense_ffn, sparse_ffn_sequential) run on the
GPU through the C ABI; the metric definitions are the reference's: "truly
active" means a strictly positive gate pre-activation (f64, the caller's
weights), recall averages over tokens with at least one truly active neuron,
the ROC AUC pools (predictor value, label) pairs over all neurons and tokens
(midrank statistic, vacuously 1 with a single class), and the output error is
||y_dense - y_sparse|| / ||y_dense|| averaged over tokens with y_dense != 0.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .ffn_exec import (DataError, FfnWeights, Predictor, dense_ffn, predict_mask,
                       sparse_ffn_sequential, validate_predictor, validate_weights)


def roc_auc(scores, labels) -> float:
    """analysis.hpp:197-238: P(random positive outranks random negative), ties 1/2."""
    scores = np.asarray(scores, dtype=np.float64).reshape(-1)
    labels = np.asarray(labels).reshape(-1).astype(bool)
    if scores.size != labels.size:
        raise DataError("roc auc: score and label counts differ")
    pos = int(labels.sum())
    neg = labels.size - pos
    if pos == 0 or neg == 0:
        raise DataError("roc auc: need at least one positive and one negative label")
    order = np.argsort(scores, kind="stable")
    s = scores[order]
    # midranks: equal scores share the mean of their 1-based rank range
    starts = np.r_[0, np.nonzero(np.diff(s))[0] + 1]
    ends = np.r_[starts[1:], s.size]
    mid = 0.5 * ((starts + 1) + ends)
    rank = np.repeat(mid, ends - starts)
    prs = float(rank[labels[order]].sum())
    u = prs - pos * (pos + 1.0) / 2.0
    return u / (pos * float(neg))


@dataclass
class MetricRow:  # analysis.hpp:241-248
    layer: int = 0
    recall: float = 0.0
    predicted_sparsity: float = 0.0
    realized_sparsity: float = 0.0
    roc_auc: float = 0.0
    mean_rel_output_error: float = 0.0


def layer_metrics(w: FfnWeights, pred: Predictor, x_cols, layer: int = 0) -> MetricRow:
    """analysis.hpp:250-326 with the executor on the GPU. x_cols: d x T (tokens as columns)."""
    validate_weights(w)
    validate_predictor(pred)
    X = np.asarray(x_cols, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] < 1:
        raise DataError("activation batch: need at least one token")
    if not np.all(np.isfinite(X)):
        raise DataError("activation batch: non-finite entries")
    if X.shape[0] != w.hidden_size() or pred.inter_size() != w.inter_size() or \
            pred.hidden_size() != w.hidden_size():
        raise DataError("layer metrics: shapes disagree")
    T = X.shape[1]
    row = MetricRow(layer=layer)
    gate_pre = w.gate @ X                              # labels: truly active (f64)
    pred_pre = pred.A @ (pred.B @ X) + pred.bias[:, None]  # scores
    recall_sum, recall_tokens, err_sum, err_tokens = 0.0, 0, 0.0, 0
    for t in range(T):
        x = X[:, t]
        mask = predict_mask(pred, x).active.astype(bool)
        active = gate_pre[:, t] > 0.0
        if active.any():
            recall_sum += float((mask & active).sum()) / float(active.sum())
            recall_tokens += 1
        dense = dense_ffn(w, x)
        sparse = sparse_ffn_sequential(w, pred, x)
        row.predicted_sparsity += sparse.stats.predicted_sparsity
        row.realized_sparsity += sparse.stats.realized_sparsity
        dn = float(np.linalg.norm(dense.y))
        if dn > 0.0:
            err_sum += float(np.linalg.norm(dense.y - sparse.y)) / dn
            err_tokens += 1
    row.recall = recall_sum / recall_tokens if recall_tokens else 1.0
    row.predicted_sparsity /= T
    row.realized_sparsity /= T
    row.mean_rel_output_error = err_sum / err_tokens if err_tokens else 0.0
    labels = gate_pre > 0.0
    row.roc_auc = roc_auc(pred_pre, labels) if labels.any() and not labels.all() else 1.0
    return row


# ---- the cmd_run JSONL parity stream ----
def fnv1a64(data: bytes) -> int:
    """sparsegate_main.cpp:73-81: FNV-1a 64 over raw bytes, with the reference's offset
    basis literal 1469598103934665603 (not the published 14695981039346656037) so that
    hashes match the reference's streams."""
    h = 1469598103934665603
    for b in bytes(data):
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def hex64(v: int) -> str:  # sparsegate_main.cpp:83-87 ("%016" PRIx64)
    return f"{v & 0xFFFFFFFFFFFFFFFF:016x}"


def run_record(t: int, result) -> dict:
    """One cmd_run record (sparsegate_main.cpp:251-258) for token t: the executor's stats
    and the FNV-1a hash of y as f64 bytes."""
    y = np.ascontiguousarray(np.asarray(result.y, dtype="<f8"))
    return {"token_index": int(t),
            "predicted_sparsity": float(result.stats.predicted_sparsity),
            "realized_sparsity": float(result.stats.realized_sparsity),
            "multiplies": int(result.stats.multiplies),
            "output_hash": hex64(fnv1a64(y.tobytes()))}


def format_stream(records) -> str:
    """JSONL as cmd_run writes it: one compact object per line, keys in nlohmann's
    (std::map) order, shortest round-trip doubles."""
    import json
    return "".join(json.dumps(r, sort_keys=True, separators=(",", ":")) + "\n" for r in records)


def run_stream(w: FfnWeights, pred, x_cols, mode: str = "sequential") -> str:
    """cmd_run (sparsegate_main.cpp:224-267) with the executor on the GPU: mode dense,
    parallel or sequential over the tokens (columns) of x_cols. The stats fields equal
    the reference's whenever the index sets do; output_hash hashes the GPU's y (fp32
    widened to f64), so it is stable run to run but not equal to the f64 CPU hash."""
    from .ffn_exec import sparse_ffn_parallel
    X = np.asarray(x_cols, dtype=np.float64)
    if X.ndim != 2:
        raise DataError("activation batch: expected d x tokens")
    recs = []
    for t in range(X.shape[1]):
        x = X[:, t]
        if mode == "dense":
            r = dense_ffn(w, x)
        elif mode == "parallel":
            r = sparse_ffn_parallel(w, pred, x)
        elif mode == "sequential":
            r = sparse_ffn_sequential(w, pred, x)
        else:
            raise DataError(f"unknown mode {mode}")
        recs.append(run_record(t, r))
    return format_stream(recs)
