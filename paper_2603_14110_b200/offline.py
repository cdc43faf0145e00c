"""Offline producer of the executor's predictor (host only, not on the decode path).

Restates the reference's offline stages, which the north star keeps on the host:
  * ``cholesky_whitening``  factorization.hpp:31-59  (damping ladder {0,1,10,100}·1e-10·μ)
  * ``build_predictor``     factorization.hpp:93-144 (A = U_r Σ_r, B = V_rᵀ S⁻¹, bias 0)
  * ``proxy_scores``        calibration.hpp:39-46    (A (B X))
  * ``damage_weights``      calibration.hpp:20-36
  * ``greedy_calibrate``    calibration.hpp:61-205   (C++ in libsparsegate_b200.so)

The dense linear algebra (Gram, Cholesky, SVD) uses numpy/LAPACK in f64 as the
reference uses Eigen; ``svd="randomized"`` swaps the exact thin SVD for a
seeded randomized range finder (Halko et al.) so bench-size predictors build in
seconds — the bench states which one it used.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi as capi
from .ffn_exec import Activation, DataError, FfnWeights, Predictor, check


@dataclass
class BuildResult:
    predictor: Predictor
    singular_values: np.ndarray
    lam: float = 0.0
    mode: str = "whitened"


def cholesky_whitening(X: np.ndarray, epsilon: float = 1e-10,
                       multipliers=(0.0, 1.0, 10.0, 100.0)):
    """factorization.hpp:31-59. X: d x n (tokens as columns). Returns (S, S_inv, λ)."""
    if X.shape[1] < 1:
        raise DataError("activation batch: need at least one token")
    if not np.all(np.isfinite(X)):
        raise DataError("activation batch: non-finite entries")
    d = X.shape[0]
    gram = X @ X.T
    mu = np.trace(gram) / d
    tried = []
    for m in multipliers:
        lam = m * epsilon * mu
        try:
            S = np.linalg.cholesky(gram + lam * np.eye(d))
        except np.linalg.LinAlgError:
            tried.append(lam)
            continue
        import scipy.linalg as sla
        S_inv = sla.solve_triangular(S, np.eye(d), lower=True)
        return S, S_inv, lam
    raise DataError("cholesky whitening failed for every damping value {"
                    + ", ".join(f"{t:g}" for t in tried) + "}; calibration data is degenerate")


def _randomized_svd(M: np.ndarray, k: int, oversample: int = 16, power_iters: int = 2,
                    seed: int = 0):
    rng = np.random.default_rng(seed)
    m, n = M.shape
    ell = min(n, k + oversample)
    Q, _ = np.linalg.qr(M @ rng.standard_normal((n, ell)))
    for _ in range(power_iters):
        Q, _ = np.linalg.qr(M.T @ Q)
        Q, _ = np.linalg.qr(M @ Q)
    Bs = Q.T @ M
    Ub, s, Vt = np.linalg.svd(Bs, full_matrices=False)
    return Q @ Ub[:, :k], s[:k], Vt[:k]


def build_predictor(w_gate: np.ndarray, X: np.ndarray, rank: int, mode: str = "whitened",
                    svd: str = "exact", seed: int = 0) -> BuildResult:
    """factorization.hpp:93-144."""
    D, d = w_gate.shape
    if rank < 1 or rank > min(D, d):
        raise DataError(f"predictor rank {rank} out of range [1, {min(D, d)}]")
    if not np.all(np.isfinite(w_gate)):
        raise DataError("gate matrix has non-finite entries")
    lam = 0.0
    if mode == "whitened":
        if X.shape[0] != d:
            raise DataError(f"calibration batch hidden size {X.shape[0]} does not match gate "
                            f"columns {d}")
        S, S_inv, lam = cholesky_whitening(X)
        target = w_gate @ S
    else:
        target = w_gate
    if svd == "exact":
        U, s, Vt = np.linalg.svd(target, full_matrices=False)
        U, s_r, Vt = U[:, :rank], s[:rank], Vt[:rank]
    else:
        U, s_r, Vt = _randomized_svd(target, rank, seed=seed)
        s = s_r
    A = U * s_r[None, :]
    B = Vt @ S_inv if mode == "whitened" else Vt.copy()
    return BuildResult(Predictor(np.ascontiguousarray(A), np.ascontiguousarray(B), np.zeros(D),
                                 rank), s, lam, mode)


def proxy_scores(pred: Predictor, X: np.ndarray) -> np.ndarray:
    """calibration.hpp:39-46: s_i(t) = (A (B x_t))_i, D x T."""
    return pred.A @ (pred.B @ X)


def damage_weights(w: FfnWeights, X: np.ndarray) -> np.ndarray:
    """calibration.hpp:20-36: |act(gate·x)·up_factor|² · ‖down_col_i‖², D x T."""
    gp = w.gate @ X
    upre = w.up @ X
    if w.activation == Activation.DReLU:
        inner = np.maximum(gp, 0.0) * np.maximum(upre, 0.0)
    else:
        inner = np.maximum(gp, 0.0) * upre
    down_norm2 = np.sum(w.down * w.down, axis=0)
    return inner * inner * down_norm2[:, None]


@dataclass
class CalibResult:
    bias: np.ndarray
    achieved_sparsity: float
    total_damage: float


def greedy_calibrate(scores: np.ndarray, weights: np.ndarray, eta: int = 8,
                     target_sparsity: float = 0.5) -> CalibResult:
    """calibration.hpp:61-96 + :128-205 (bias = -τ, +inf where nothing is dropped)."""
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    if scores.shape != weights.shape:
        raise DataError("calibration instance: score and weight shapes differ")
    D, T = scores.shape
    bias = np.zeros(D)
    ach, dmg = C.c_double(0), C.c_double(0)
    check(capi.lib().sg_greedy_calibrate(scores.ctypes.data_as(C.c_void_p),
                                         weights.ctypes.data_as(C.c_void_p), D, T, eta,
                                         target_sparsity, bias.ctypes.data_as(C.c_void_p),
                                         C.byref(ach), C.byref(dmg)))
    return CalibResult(bias, ach.value, dmg.value)
