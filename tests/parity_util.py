"""Parity rules shared by the GPU tests.

* Inputs: the GPU uploads weights rounded f64 -> f32 -> bf16 (RNE); the oracle
  runs in f64 on exactly those rounded values widened back to f64 (and on the
  fp32-rounded bias / x), so rounding of the inputs is never counted as error.
* Index sets (integer work) must be bit-exact, except neurons whose f64
  pre-activation lies within EPS of the decision threshold relative to its
  absolute-value scale:  |pre_i| <= EPS * (sum_j |A_ij| sum_k |B_jk x_k| + |b_i|)
  for P, |g_i| <= EPS * sum_k |gate_ik x_k| for V.  EPS = 2^-14 bounds fp32
  accumulation (one rounding per FMA, <= d/32 + 5 + 16 chained roundings per dot
  for d <= 32768) with margin.
* y (fp32 accumulation, fp32 output) must satisfy
  ||y_gpu - y_ref||_2 <= Y_RTOL * ||y_ref||_2 with Y_RTOL = 1e-3, where y_ref is
  the oracle output; when a token's sets differ (only at admissible neurons)
  y_ref is recomputed in f64 on the GPU's own sets.
* The number of such admissible flips is bounded: at most MAX_FLIPS neurons
  per token may differ in P, and as many in V (observed: 0 on almost every
  token; tests record the counts and the band sizes).
"""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_2603_14110_b200 import bf16_to_f64, round_bf16

EPS = 2.0 ** -14
Y_RTOL = 1e-3
MAX_FLIPS = 4


def q_bf16(a) -> np.ndarray:
    """The values the GPU computes with: f64 -> f32 -> bf16 -> f64."""
    return bf16_to_f64(round_bf16(a))


def q_f32(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def quantize_layer(gate, up, down, A=None, B=None, bias=None):
    out = dict(gate=q_bf16(gate), up=q_bf16(up), down=q_bf16(down))
    if A is not None:
        out.update(A=q_bf16(A), B=q_bf16(B), bias=q_f32(bias))
    return out


def gated(g, u, act):
    z = np.where(g > 0, g * u, 0.0)
    if act == 1:
        z = np.where(u > 0, z, 0.0)
    return z


def check_token(q, x, gpu_y, gpu_P, gpu_V, act=0, eps=EPS, y_rtol=Y_RTOL, max_flips=MAX_FLIPS,
                y_atol=0.0):
    """Compare one GPU token with the oracle. q: quantized layer dict (f64).

    Returns a dict of diagnostics; raises AssertionError on a parity failure.
    """
    xq = q_f32(x)
    o = O.sparse_ffn(q["gate"], q["up"], q["down"], q["A"], q["B"], q["bias"], xq, activation=act)
    mask, cnt, pre = O.predict_mask(q["A"], q["B"], q["bias"], xq)
    ps, gs = O.threshold_scales(q["A"], q["B"], q["bias"], q["gate"], xq)
    D = q["gate"].shape[0]
    near_p = np.abs(pre) <= eps * ps
    gfull = q["gate"] @ xq
    near_v = np.abs(gfull) <= eps * gs
    P_ref, V_ref = set(o.P.tolist()), set(o.V.tolist())
    P_gpu, V_gpu = set(np.asarray(gpu_P).tolist()), set(np.asarray(gpu_V).tolist())
    dP = P_ref ^ P_gpu
    bad_P = [i for i in dP if not near_p[i]]
    assert not bad_P, f"P differs outside the near-threshold band at {bad_P[:10]}"
    # V must equal {i in P_gpu : g_i > 0} up to near-threshold gate neurons
    dV = V_gpu ^ {i for i in P_gpu if gfull[i] > 0}
    bad_V = [i for i in dV if not near_v[i]]
    assert not bad_V, f"V differs outside the near-threshold band at {bad_V[:10]}"
    assert len(dP) <= max_flips and len(dV) <= max_flips, \
        f"{len(dP)} P / {len(dV)} V near-threshold flips exceed the bound {max_flips}"
    assert len(gpu_P) == len(P_gpu) and list(gpu_P) == sorted(gpu_P), "P not ascending/unique"
    assert len(gpu_V) == len(V_gpu) and list(gpu_V) == sorted(gpu_V), "V not ascending/unique"
    if not dP and not dV:
        assert V_gpu == V_ref
        y_ref = o.y
    else:
        idx = np.array(sorted(V_gpu), dtype=np.int64)
        u = q["up"][idx] @ xq
        z = gated(gfull[idx], u, act)
        y_ref = q["down"][:, idx] @ z
    gpu_y = np.asarray(gpu_y, dtype=np.float64)
    nrm = np.linalg.norm(y_ref)
    err = np.linalg.norm(gpu_y - y_ref)
    if nrm == 0:
        assert err <= y_atol, f"expected exact zero output, got |y|={err}"
        rel = 0.0
    elif err <= y_atol:
        rel = 0.0
    else:
        rel = err / nrm
        assert rel <= y_rtol, f"y relative error {rel:.3e} > {y_rtol}"
    return dict(rel=rel, p=len(P_gpu), v=len(V_gpu), dP=len(dP), dV=len(dV),
                near_p=int(near_p.sum()), near_v=int(near_v.sum()), oracle=o)
