"""Multi-layer synthetic decode models for the bench (host-side setup only).

A "model" is a stack of L sparse-FFN layers of one BASELINE.json shape, each
built exactly as SURVEY.md §8(d) prescribes:
  * weights: make_synthetic_fixture{hidden=d, inter=D, natural_sparsity=0.9,
    activation, seed=base+ℓ} (synthetic.hpp:80-108), emitted as bf16 with
    `down` neuron-major;
  * predictor: rank-r truncated SVD of W_gate (naive mode, factorization.hpp:93-144
    with S = I) by a seeded randomized range finder, then greedy bias
    calibration (calibration.hpp:61-205) on the fixture's calibration tokens to
    predicted sparsity s, η = 8;
  * input token of layer ℓ: eval token 0 of layer ℓ's fixture (N(1,1), bf16-exact).
None of this is timed; it produces the resident inputs of the timed executor.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
from dataclasses import dataclass

import numpy as np

from .ffn_exec import Activation, DeviceLayer, bf16_to_f64, round_bf16
from .offline import _randomized_svd, greedy_calibrate
from .synthetic import SyntheticConfig, make_synthetic_bf16

CONFIGS = {
    # BASELINE.json configs[0]: one 7B-shape layer (the CPU-reference case)
    "1layer": dict(d=4096, D=11008, L=1, act=0, model="single ReGLU FFN layer d=4096 d_ff=11008"),
    # configs[1]: the headline
    "7b": dict(d=4096, D=11008, L=32, act=0, model="ProSparse-Llama2-7B FFN stack"),
    # configs[2]
    "mistral": dict(d=4096, D=14336, L=32, act=1, model="TurboSparse-Mistral-7B FFN stack (dReLU)"),
    # configs[3]
    "13b": dict(d=5120, D=13824, L=40, act=0, model="ProSparse-Llama2-13B FFN stack"),
    # small, for smoke tests
    "tiny": dict(d=512, D=1408, L=4, act=0, model="tiny test stack"),
}


@dataclass
class HostLayer:
    gate: np.ndarray   # uint16 D x d
    up: np.ndarray     # uint16 D x d
    down_t: np.ndarray # uint16 D x d (neuron-major)
    A: np.ndarray      # uint16 D x r
    B: np.ndarray      # uint16 r x d
    bias: np.ndarray   # f64 D (+inf allowed)
    x: np.ndarray      # f64 d (eval token 0), bf16-exact
    xs: np.ndarray     # f64 d x T eval tokens
    calib_achieved: float = 0.0
    load: np.ndarray = None  # expected rows streamed per token per neuron (calibration stats)


def build_host_layer(d, D, act, seed, rank=256, sparsity=0.5, calib_tokens=256, eval_tokens=16,
                     eta=8, power_iters=1) -> HostLayer:
    fx = make_synthetic_bf16(SyntheticConfig(hidden=d, inter=D, calib_tokens=calib_tokens,
                                             eval_tokens=eval_tokens, activation=Activation(act),
                                             seed=seed))
    G = bf16_to_f64(fx["gate"]).astype(np.float32)
    U, s, Vt = _randomized_svd(G, rank, oversample=8, power_iters=power_iters, seed=seed)
    A = (U * s[None, :]).astype(np.float64)
    B = Vt.astype(np.float64)
    # the executor sees bf16 factors; calibrate the bias on exactly those
    Aq = bf16_to_f64(round_bf16(A)).astype(np.float32)
    Bq = bf16_to_f64(round_bf16(B)).astype(np.float32)
    Xc = bf16_to_f64(round_bf16(fx["calib"])).astype(np.float32)
    scores = (Aq @ (Bq @ Xc)).astype(np.float64)
    gp = G @ Xc
    up = bf16_to_f64(fx["up"]).astype(np.float32) @ Xc
    if act == 1:
        inner = np.maximum(gp, 0) * np.maximum(up, 0)
    else:
        inner = np.maximum(gp, 0) * up
    dn = bf16_to_f64(fx["down_t"])
    down_norm2 = np.sum(dn * dn, axis=1)
    weights = (inner.astype(np.float64) ** 2) * down_norm2[:, None]
    cal = greedy_calibrate(scores, weights, eta, sparsity)
    ev = bf16_to_f64(round_bf16(fx["eval"]))
    # offline activity statistics of the calibrated predictor on the calibration
    # tokens: a neuron costs one gate row when predicted active and two more rows
    # (up, down) when it also survives revalidation
    on = (scores + cal.bias[:, None].astype(np.float32)) > 0
    load = on.mean(axis=1) + 2.0 * (on & (gp > 0)).mean(axis=1)
    return HostLayer(fx["gate"], fx["up"], fx["down_t"], round_bf16(A), round_bf16(B), cal.bias,
                     ev[:, 0].copy(), ev, cal.achieved_sparsity, load)


def build_host_model(config: str, layers: int = None, seed_base: int = 0, rank: int = 256,
                     sparsity: float = 0.5, workers: int = None, log=None, eval_tokens: int = 16):
    cfg = CONFIGS[config]
    L = layers or cfg["L"]
    workers = workers or max(1, min(L, (os.cpu_count() or 4) // 2))
    out = [None] * L
    with cf.ThreadPoolExecutor(workers) as ex:
        futs = {ex.submit(build_host_layer, cfg["d"], cfg["D"], cfg["act"], seed_base + l, rank,
                          sparsity, eval_tokens=eval_tokens): l for l in range(L)}
        for f in cf.as_completed(futs):
            out[futs[f]] = f.result()
            if log:
                log(f"layer {futs[f]} ready")
    return cfg, out


def balanced_order(load: np.ndarray, neurons: np.ndarray, G: int) -> np.ndarray:
    """Layout order of `neurons` for G CTAs: CTA c gets the c-th contiguous block of
    the layout (sizes c*n/G boundaries, as the kernel splits), and blocks get equal
    expected load: neurons by decreasing load are dealt to the CTAs in serpentine
    order (skipping full ones). Deterministic; within a block by decreasing load
    (ties ascending), so each block's most frequently predicted neurons lead it
    (the hot prefix of sg_layer_set_hot_rows)."""
    n = len(neurons)
    bounds = [c * n // G for c in range(G + 1)]
    cap = np.diff(bounds)
    bins = [[] for _ in range(G)]
    order = neurons[np.argsort(-load[neurons], kind="stable")]
    c, step = 0, 1
    for nid in order:
        while len(bins[c]) >= cap[c]:
            c += step
            if c == G or c < 0:
                step = -step
                c += step
        bins[c].append(nid)
        c += step
        if c == G or c < 0:
            step = -step
            c += step
    out = []
    for b in bins:
        b = np.sort(np.asarray(b, dtype=np.int64))
        out.append(b[np.argsort(-load[b], kind="stable")])
    return np.concatenate(out)


def upload(host: HostLayer, d, D, act, rank=256, device=0, shard_index=0, shard_count=1,
           balance=True, hot_rows=16):
    """Device layer of a host layer. balance=True: the single-token executor's
    per-CTA load-balanced neuron layout (balanced_order); "sorted": neurons by
    decreasing calibration activity, so a batch's survivor rows gather into the
    leading blocks and the trailing blocks' down rows are skipped whole
    (csrc/sg_batch_tc.cu); False: ascending."""
    raw = dict(hidden=d, inter=D, rank=rank, activation=act, gate=host.gate, up=host.up,
               down_t=host.down_t, A=host.A, B=host.B, bias=host.bias)
    if balance == "sorted" and host.load is not None:
        raw["order"] = np.argsort(-host.load, kind="stable").astype(np.int64)
        balance = False
    if balance and host.load is not None:
        import torch
        from .sharded import shard_indices
        G = torch.cuda.get_device_properties(device).multi_processor_count
        mine = shard_indices(D, shard_index, shard_count)
        first = balanced_order(host.load, mine, G)
        rest = np.setdiff1d(np.arange(D, dtype=np.int64), mine)
        raw["order"] = np.concatenate([first, rest])
    layer = DeviceLayer(raw=raw, device=device, shard_index=shard_index, shard_count=shard_count)
    if balance and host.load is not None and hot_rows:
        layer.set_hot_rows(hot_rows)
    return layer
