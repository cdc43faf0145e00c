"""The C++ offline producer (csrc/sg_offline.cu) against the numpy
restatement of factorization.hpp / calibration.hpp (paper_2603_14110_b200/offline.py):
Cholesky whitening, the exact (Jacobi) and randomized (GPU) predictor builds, proxy
scores and damage weights."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_14110_b200 import _capi as capi
from paper_2603_14110_b200 import offline
from paper_2603_14110_b200.ffn_exec import DataError, check
from paper_2603_14110_b200.synthetic import SyntheticConfig, make_synthetic_fixture

pytestmark = pytest.mark.gpu
_D = C.c_double


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _native_build(W, X, r, whitened, mode, n_sv):
    D, d = W.shape
    W = np.ascontiguousarray(W, dtype=np.float64)
    Xc = np.ascontiguousarray(X, dtype=np.float64) if X is not None else None
    A = np.zeros((D, r))
    B = np.zeros((r, d))
    sv = np.zeros(n_sv)
    mult = np.array([0.0, 1.0, 10.0, 100.0])
    s1, lam = _D(0), _D(0)
    check(capi.lib().sg_build_predictor(_p(W), D, d, _p(Xc) if Xc is not None else None,
                                        0 if Xc is None else Xc.shape[1], r, int(whitened), mode, 7,
                                        1e-10, _p(mult), 4, _p(A), _p(B), _p(sv), n_sv, C.byref(s1),
                                        C.byref(lam)))
    return A, B, sv, s1.value, lam.value


@pytest.mark.parametrize("whitened", [False, True])
def test_exact_build_matches_numpy(whitened):
    fx = make_synthetic_fixture(SyntheticConfig(hidden=64, inter=256, calib_tokens=512, eval_tokens=2, seed=3))
    W, X, r = fx.weights.gate, fx.calib, 16
    ref = offline.build_predictor(W, X, r, mode="whitened" if whitened else "naive", svd="exact")
    A, B, sv, s1, lam = _native_build(W, X, r, whitened, 0, 64)
    pr = ref.predictor
    # factors are unique up to the sign of each singular pair: compare A B and the spectrum
    assert np.allclose(A @ B, pr.A @ pr.B, rtol=1e-9, atol=1e-9 * np.abs(pr.A @ pr.B).max())
    assert np.allclose(sv, ref.singular_values[:64], rtol=1e-9)
    assert lam == pytest.approx(ref.lam, rel=1e-12, abs=0.0)
    w_sv = np.linalg.svd(W, compute_uv=False)
    assert s1 == pytest.approx(w_sv[r], rel=1e-9)


def test_randomized_build_on_a_7b_shape_slice():
    """The bench's naive-mode rank-256 predictor of a 2048 x 4096 gate slice through the
    GPU range finder: the captured spectrum and the residual match the exact SVD."""
    rng = np.random.default_rng(0)
    D, d, r = 2048, 4096, 256
    U = np.linalg.qr(rng.standard_normal((D, 300)))[0]
    V = np.linalg.qr(rng.standard_normal((d, 300)))[0]
    s = np.exp(-np.arange(300) / 40.0)
    W = (U * s) @ V.T + 1e-4 * rng.standard_normal((D, d))
    A, B, sv, s1, _ = _native_build(W, None, r, False, 1, r)
    ex = np.linalg.svd(W, compute_uv=False)
    # above the noise floor (sigma ~ 1e-2 here) the spectrum is exact; at the flat
    # floor a range finder of width r + 32 with 4 power iterations stays within a few %
    assert np.allclose(sv[:128], ex[:128], rtol=1e-6)
    assert np.allclose(sv[:r], ex[:r], rtol=0.08)
    res = np.linalg.norm(W - A @ B, 2)
    assert res <= 1.06 * ex[r]


def test_whitening_and_calibration_inputs_match_numpy():
    fx = make_synthetic_fixture(SyntheticConfig(hidden=96, inter=320, calib_tokens=400, eval_tokens=2, seed=5))
    X = np.ascontiguousarray(fx.calib)
    d, T = X.shape
    S = np.zeros((d, d))
    Si = np.zeros((d, d))
    lam = _D(0)
    mult = np.array([0.0, 1.0, 10.0, 100.0])
    check(capi.lib().sg_cholesky_whitening(_p(X), d, T, 1e-10, _p(mult), 4, _p(S), _p(Si), C.byref(lam)))
    S_ref, Si_ref, lam_ref = offline.cholesky_whitening(X)
    assert np.allclose(S, S_ref, rtol=1e-10, atol=1e-10 * np.abs(S_ref).max())
    assert np.allclose(Si, Si_ref, rtol=1e-8, atol=1e-8 * np.abs(Si_ref).max())
    pred = offline.build_predictor(fx.weights.gate, X, 12, svd="exact").predictor
    D, r = pred.A.shape
    sc = np.zeros((D, T))
    check(capi.lib().sg_proxy_scores(_p(np.ascontiguousarray(pred.A)), _p(np.ascontiguousarray(pred.B)), D, r, d,
                                     _p(X), T, _p(sc)))
    assert np.allclose(sc, offline.proxy_scores(pred, X), rtol=1e-10, atol=1e-10)
    for act in (0, 1):
        w = fx.weights
        w.activation = act
        dw = np.zeros((D, T))
        check(capi.lib().sg_damage_weights(_p(np.ascontiguousarray(w.gate)), _p(np.ascontiguousarray(w.up)),
                                           _p(np.ascontiguousarray(w.down)), D, d, act, _p(X), T, _p(dw)))
        ref = offline.damage_weights(w, X)
        assert np.allclose(dw, ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max())


def test_offline_errors():
    W = np.ones((8, 4))
    W[1, 1] = np.nan
    A, B, sv = np.zeros((8, 2)), np.zeros((2, 4)), np.zeros(2)
    s1, lam = _D(0), _D(0)
    with pytest.raises(DataError):
        check(capi.lib().sg_build_predictor(_p(W), 8, 4, None, 0, 2, 0, 0, 0, 1e-10, None, 0, _p(A), _p(B),
                                            _p(sv), 2, C.byref(s1), C.byref(lam)))
    W[1, 1] = 0.0
    with pytest.raises(DataError):
        check(capi.lib().sg_build_predictor(_p(W), 8, 4, None, 0, 5, 0, 0, 0, 1e-10, None, 0, _p(A), _p(B),
                                            _p(sv), 2, C.byref(s1), C.byref(lam)))
    X = np.zeros((4, 3))  # degenerate: every damping rung fails
    S = np.zeros((4, 4))
    mult = np.array([0.0, 1.0, 10.0, 100.0])
    with pytest.raises(DataError):
        check(capi.lib().sg_cholesky_whitening(_p(X), 4, 3, 1e-10, _p(mult), 4, _p(S), _p(S), C.byref(lam)))
