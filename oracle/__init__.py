"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

ctypes bindings for
  * ``oracle/liboracle.so``  — the f64 CPU restatement of the reference executor
    (``oracle/sg_oracle.cpp``; follows /root/reference/proj/include/sparsegate/
    ffn_exec.hpp:56-244, common.hpp:52-95, synthetic.hpp:15-108), and
  * ``oracle/_ref/libsgref.so`` — the reference's own headers compiled
    unmodified (``oracle/ref_driver.cpp``), present wherever it was built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module. The product package
``paper_2603_14110_b200`` must never import it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libsgref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class Stats(C.Structure):
    _fields_ = [
        ("predicted_sparsity", C.c_double),
        ("realized_sparsity", C.c_double),
        ("multiplies", C.c_int64),
        ("pipeline", C.c_int32),
        ("pad", C.c_int32),
    ]


def build(force: bool = False) -> None:
    """Compile the restatement (and _ref when /root/reference exists)."""
    if force or not os.path.exists(LIB_PATH) or (
        os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "sg_oracle.cpp"))
    ):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    elif os.path.isdir("/root/reference/proj/include/sparsegate") and not os.path.exists(REF_PATH):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB_PATH)
        _lib.sgo_last_error.restype = C.c_char_p
        _lib.sgo_det_dot.restype = C.c_double
        _lib.sgo_det_sum.restype = C.c_double
        _lib.sgo_normal_quantile.restype = C.c_double
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The real reference executor (oracle/_ref). Raises if it was never built."""
    global _ref
    if _ref is None:
        if not ref_available():
            build()
        if not ref_available():
            raise FileNotFoundError("oracle/_ref/libsgref.so not built (needs /root/reference)")
        _ref = C.CDLL(REF_PATH)
        _ref.sgref_last_error.restype = C.c_char_p
        _ref.sgref_rng_new.restype = C.c_void_p
        _ref.sgref_rng_new.argtypes = [C.c_uint64]
        _ref.sgref_rng_free.argtypes = [C.c_void_p]
        _ref.sgref_random_matrix.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_double, _dp]
        _ref.sgref_random_gaussian.argtypes = [
            C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_double, _dp]
        _ref.sgref_uniform.restype = C.c_double
        _ref.sgref_uniform.argtypes = [C.c_void_p, C.c_double, C.c_double]
        _ref.sgref_det_dot.restype = C.c_double
        _ref.sgref_det_sum.restype = C.c_double
        _ref.sgref_normal_quantile.restype = C.c_double
        _ref.sgref_normal_quantile.argtypes = [C.c_double]
        _ref.sgref_layer_new.restype = C.c_void_p
        _ref.sgref_layer_free.argtypes = [C.c_void_p]
        _ref.sgref_thread_budget.restype = C.c_uint
    return _ref


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int, which) -> None:
    if rc != 0:
        msg = (which.sgo_last_error() if hasattr(which, "sgo_last_error")
               else which.sgref_last_error())
        raise OracleError(rc, msg.decode())


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# Restatement (liboracle.so)
# ---------------------------------------------------------------------------
@dataclass
class SparseOut:
    y: np.ndarray
    stats: Stats
    P: np.ndarray  # int32 ascending predicted-active indices
    V: np.ndarray  # int32 ascending gate-revalidated survivors
    g: np.ndarray  # gate pre-activations over P
    z: np.ndarray  # gated values over P


def det_dot(a, b) -> float:
    a, b = _c(a), _c(b)
    return lib().sgo_det_dot(_p(a), _p(b), C.c_int64(a.size))


def det_sum(v) -> float:
    v = _c(v)
    return lib().sgo_det_sum(_p(v), C.c_int64(v.size))


def dense_ffn(gate, up, down, x, activation: int = 0, scan: bool = True):
    """ffn_exec.hpp:103-122. gate/up: D x d, down: d x D (reference layout)."""
    gate, up, down, x = _c(gate), _c(up), _c(down), _c(x)
    D, d = gate.shape
    y = np.zeros(d)
    st = Stats()
    _check(lib().sgo_dense_ffn(C.c_int64(d), C.c_int64(D), C.c_int(activation), _p(gate), _p(up),
                               _p(down), _p(x), C.c_int64(x.size), C.c_int(int(scan)), _p(y),
                               C.byref(st)), lib())
    return y, st


def predict_mask(A, B, bias, x, rank_field=None):
    """ffn_exec.hpp:125-146 -> (mask uint8[D], count, pre f64[D])."""
    A, B, bias, x = _c(A), _c(B), _c(bias), _c(x)
    D, r = A.shape
    d = B.shape[1]
    mask = np.zeros(D, dtype=np.uint8)
    pre = np.zeros(D)
    cnt = C.c_int64(0)
    _check(lib().sgo_predict_mask(C.c_int64(d), C.c_int64(D), C.c_int64(r),
                                  C.c_int64(r if rank_field is None else rank_field), _p(A), _p(B),
                                  _p(bias), _p(x), C.c_int64(x.size), _p(mask), C.byref(cnt),
                                  _p(pre)), lib())
    return mask, cnt.value, pre


def sparse_ffn(gate, up, down, A, B, bias, x, activation: int = 0, pipeline: int = 2,
               scan: bool = True, rank_field=None) -> SparseOut:
    """ffn_exec.hpp:149-218 (pipeline 1 parallel, 2 sequential) + P, V, g, z."""
    gate, up, down, A, B, bias, x = map(_c, (gate, up, down, A, B, bias, x))
    D, d = gate.shape
    r = A.shape[1]
    y = np.zeros(d)
    st = Stats()
    P = np.zeros(D, dtype=np.int32)
    V = np.zeros(D, dtype=np.int32)
    g = np.zeros(D)
    z = np.zeros(D)
    p = C.c_int64(0)
    v = C.c_int64(0)
    _check(lib().sgo_sparse_ffn(
        C.c_int(pipeline), C.c_int64(d), C.c_int64(D), C.c_int(activation), _p(gate), _p(up),
        _p(down), C.c_int64(r), C.c_int64(r if rank_field is None else rank_field), _p(A), _p(B),
        _p(bias), _p(x), C.c_int64(x.size), C.c_int(int(scan)), _p(y), C.byref(st), _p(P),
        C.byref(p), _p(V), C.byref(v), _p(g), _p(z)), lib())
    return SparseOut(y, st, P[: p.value].copy(), V[: v.value].copy(), g[: p.value].copy(),
                     z[: p.value].copy())


def threshold_scales(A, B, bias, gate, x):
    """Absolute-value scales for the near-threshold rule."""
    A, B, bias, gate, x = map(_c, (A, B, bias, gate, x))
    D, r = A.shape
    d = B.shape[1]
    ps = np.zeros(D)
    gs = np.zeros(D)
    lib().sgo_threshold_scales(C.c_int64(d), C.c_int64(D), C.c_int64(r), _p(A), _p(B), _p(bias),
                               _p(gate), _p(x), _p(ps), _p(gs))
    return ps, gs


def op_count_model(d, D, r, s, sp):
    dense = C.c_int64(0)
    sparse = C.c_double(0)
    ratio = C.c_double(0)
    _check(lib().sgo_op_count_model(C.c_int64(d), C.c_int64(D), C.c_int64(r), C.c_double(s),
                                    C.c_double(sp), C.byref(dense), C.byref(sparse),
                                    C.byref(ratio)), lib())
    return dense.value, sparse.value, ratio.value


def synthetic(hidden, inter, calib_tokens=512, eval_tokens=128, natural_sparsity=0.9, seed=0,
              want=("gate", "up", "down", "calib", "eval")):
    """synthetic.hpp:80-108 restated. Returns dict of row-major f64 arrays."""
    shapes = {"gate": (inter, hidden), "up": (inter, hidden), "down": (hidden, inter),
              "calib": (hidden, calib_tokens), "eval": (hidden, eval_tokens)}
    out = {k: (np.zeros(s) if k in want else None) for k, s in shapes.items()}
    _check(lib().sgo_synthetic(
        C.c_int64(hidden), C.c_int64(inter), C.c_int64(calib_tokens), C.c_int64(eval_tokens),
        C.c_int(0), C.c_double(natural_sparsity), C.c_uint64(seed),
        *[_p(out[k]) for k in ("gate", "up", "down", "calib", "eval")]), lib())
    return {k: v for k, v in out.items() if v is not None}


# ---------------------------------------------------------------------------
# Real reference (oracle/_ref/libsgref.so)
# ---------------------------------------------------------------------------
class RefRng:
    """A std::mt19937_64 stream driven through the reference's own helpers."""

    def __init__(self, seed: int):
        self._h = C.c_void_p(ref().sgref_rng_new(seed))

    def __del__(self):
        try:
            ref().sgref_rng_free(self._h)
        except Exception:
            pass

    def random_matrix(self, rows, cols, stddev=1.0):  # test_support.hpp:48-58
        out = np.zeros((rows, cols))
        ref().sgref_random_matrix(self._h, rows, cols, stddev, out)
        return out

    def random_vector(self, n, stddev=1.0):  # test_support.hpp:60-68
        return self.random_matrix(n, 1, stddev).reshape(n)

    def random_gaussian(self, rows, cols, mean, stddev):  # synthetic.hpp:32-42
        out = np.zeros((rows, cols))
        ref().sgref_random_gaussian(self._h, rows, cols, mean, stddev, out)
        return out

    def uniform(self, a=0.0, b=1.0):
        return ref().sgref_uniform(self._h, a, b)


def ref_synthetic(hidden, inter, calib_tokens=512, eval_tokens=128, natural_sparsity=0.9, seed=0):
    out = {"gate": np.zeros((inter, hidden)), "up": np.zeros((inter, hidden)),
           "down": np.zeros((hidden, inter)), "calib": np.zeros((hidden, calib_tokens)),
           "eval": np.zeros((hidden, eval_tokens))}
    R = ref()
    _check(R.sgref_synthetic(
        C.c_int64(hidden), C.c_int64(inter), C.c_int64(calib_tokens), C.c_int64(eval_tokens),
        C.c_int(0), C.c_double(natural_sparsity), C.c_uint64(seed),
        *[_p(out[k]) for k in ("gate", "up", "down", "calib", "eval")]), R)
    return out


def ref_greedy_calibrate(scores, weights, eta, target):
    """calibration.hpp:61-96 + :128-205 through the reference's own code: bias (D,),
    achieved sparsity, total damage."""
    scores, weights = _c(scores), _c(weights)
    D, T = scores.shape
    bias = np.zeros(D)
    ach, dmg = C.c_double(0), C.c_double(0)
    R = ref()
    R.sgref_greedy_calibrate.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                         C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
    _check(R.sgref_greedy_calibrate(_p(scores), _p(weights), C.c_int64(D), C.c_int64(T),
                                    C.c_int(eta), C.c_double(target), _p(bias), C.byref(ach),
                                    C.byref(dmg)), R)
    return bias, ach.value, dmg.value


def ref_dense_ffn(gate, up, down, x, activation=0):
    gate, up, down, x = map(_c, (gate, up, down, x))
    D, d = gate.shape
    y = np.zeros(d)
    st = Stats()
    R = ref()
    _check(R.sgref_dense_ffn(C.c_int64(d), C.c_int64(D), C.c_int(activation), _p(gate), _p(up),
                             _p(down), _p(x), C.c_int64(x.size), _p(y), C.byref(st)), R)
    return y, st


def ref_sparse_ffn(gate, up, down, A, B, bias, x, activation=0, pipeline=2, rank_field=None):
    gate, up, down, A, B, bias, x = map(_c, (gate, up, down, A, B, bias, x))
    D, d = gate.shape
    r = A.shape[1]
    y = np.zeros(d)
    st = Stats()
    R = ref()
    _check(R.sgref_sparse_ffn(
        C.c_int(pipeline), C.c_int64(d), C.c_int64(D), C.c_int(activation), _p(gate), _p(up),
        _p(down), C.c_int64(r), C.c_int64(r if rank_field is None else rank_field), _p(A), _p(B),
        _p(bias), _p(x), C.c_int64(x.size), _p(y), C.byref(st)), R)
    return y, st


def ref_predict_mask(A, B, bias, x, rank_field=None):
    A, B, bias, x = map(_c, (A, B, bias, x))
    D, r = A.shape
    d = B.shape[1]
    mask = np.zeros(D, dtype=np.uint8)
    cnt = C.c_int64(0)
    R = ref()
    _check(R.sgref_predict_mask(C.c_int64(d), C.c_int64(D), C.c_int64(r),
                                C.c_int64(r if rank_field is None else rank_field), _p(A), _p(B),
                                _p(bias), _p(x), C.c_int64(x.size), _p(mask), C.byref(cnt)), R)
    return mask, cnt.value


def ref_op_count_model(d, D, r, s, sp):
    dense = C.c_int64(0)
    sparse = C.c_double(0)
    ratio = C.c_double(0)
    R = ref()
    _check(R.sgref_op_count_model(C.c_int64(d), C.c_int64(D), C.c_int64(r), C.c_double(s),
                                  C.c_double(sp), C.byref(dense), C.byref(sparse),
                                  C.byref(ratio)), R)
    return dense.value, sparse.value, ratio.value


class RefLayer:
    """A reference FfnWeights + Predictor held in C++ for timing runs."""

    def __init__(self, gate, up, down, A=None, B=None, bias=None, activation=0):
        gate, up, down = map(_c, (gate, up, down))
        self.D, self.d = gate.shape
        r = 0 if A is None else A.shape[1]
        self._keep = [gate, up, down] + ([] if A is None else [_c(A), _c(B), _c(bias)])
        args = [C.c_int64(self.d), C.c_int64(self.D), C.c_int(activation), _p(gate), _p(up),
                _p(down), C.c_int64(r)]
        args += [None, None, None] if A is None else [_p(a) for a in self._keep[3:]]
        self._h = C.c_void_p(ref().sgref_layer_new(*args))

    def run(self, xs, pipeline=2):
        """xs: tokens x d. Returns (ys, stats list, elapsed seconds)."""
        xs = _c(xs)
        T = xs.shape[0]
        ys = np.zeros_like(xs)
        st = (Stats * T)()
        el = C.c_double(0)
        R = ref()
        _check(R.sgref_layer_run(self._h, C.c_int(pipeline), _p(xs), C.c_int64(T), _p(ys), st,
                                 C.byref(el)), R)
        return ys, list(st), el.value

    def __del__(self):
        try:
            ref().sgref_layer_free(self._h)
        except Exception:
            pass
