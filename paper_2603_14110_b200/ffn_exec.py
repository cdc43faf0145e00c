"""Host-side mirror of the reference executor API, over the C ABI.

Mirrors /root/reference/proj/include/sparsegate/ffn_exec.hpp (namespace
``sparsegate``) name for name, with the same argument meaning and error
behaviour:

=============================  ======================================  =========================
reference                      here                                    C ABI
=============================  ======================================  =========================
``dense_ffn`` :103-122         :func:`dense_ffn`                       ``sg_ffn_forward`` (DENSE)
``predict_mask`` :125-146      :func:`predict_mask`                    ``sg_predict_mask``
``sparse_ffn_parallel`` :149   :func:`sparse_ffn_parallel`             ``sg_ffn_forward`` (PARALLEL)
``sparse_ffn_sequential`` :183 :func:`sparse_ffn_sequential`           ``sg_ffn_forward`` (SEQUENTIAL)
``op_count_model`` :229-244    :func:`op_count_model`                  ``sg_op_count_model``
types ``Mask``/``ExecStats``/  same names (dataclasses)
``FfnResult``/``Pipeline``
``FfnWeights``/``Predictor``   same names (types.hpp:21-80)
errors ``DataError`` …         same names (common.hpp:20-37)
=============================  ======================================  =========================

The reference functions are stateless; the GPU needs resident weights. The
stateless functions therefore upload an ``FfnWeights``/``Predictor`` pair once
(validated once, types.hpp:31-51/:82-105) and cache the device copy keyed by
object identity — treat those objects as immutable after first use, or use
:class:`DeviceLayer` explicitly. Every computation runs on the GPU through
libsparsegate_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import threading
import weakref
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional

import numpy as np

from . import _capi as capi


# ---------------------------------------------------------------------------
# errors (common.hpp:20-37)
# ---------------------------------------------------------------------------
class Error(RuntimeError):
    pass


class IoError(Error):
    pass


class DataError(Error):
    pass


class PropertyViolation(Error):
    pass


class UsageError(Error):
    pass


class CudaError(Error):
    pass


_ERRORS = {capi.SG_ERR_USAGE: UsageError, capi.SG_ERR_DATA: DataError,
           capi.SG_ERR_PROPERTY: PropertyViolation, capi.SG_ERR_IO: IoError,
           capi.SG_ERR_CUDA: CudaError, capi.SG_ERR_NCCL: CudaError}


def check(rc: int) -> None:
    if rc != capi.SG_OK:
        msg = capi.lib().sg_last_error().decode()
        raise _ERRORS.get(rc, Error)(msg)


# ---------------------------------------------------------------------------
# types (types.hpp:12-105, ffn_exec.hpp:27-52)
# ---------------------------------------------------------------------------
class Activation(IntEnum):
    ReGLU = 0
    DReLU = 1


class Pipeline(IntEnum):
    Dense = 0
    Parallel = 1
    Sequential = 2


@dataclass(eq=False)
class FfnWeights:
    """gate, up: D x d; down: d x D (reference layout, types.hpp:19-24)."""
    gate: np.ndarray
    up: np.ndarray
    down: np.ndarray
    activation: Activation = Activation.ReGLU

    def hidden_size(self) -> int:
        return int(self.gate.shape[1])

    def inter_size(self) -> int:
        return int(self.gate.shape[0])


@dataclass(eq=False)
class Predictor:
    """A: D x r, B: r x d, bias: D (types.hpp:72-80)."""
    A: np.ndarray
    B: np.ndarray
    bias: np.ndarray
    rank: int = 0

    def hidden_size(self) -> int:
        return int(self.B.shape[1])

    def inter_size(self) -> int:
        return int(self.A.shape[0])


@dataclass
class Mask:
    active: np.ndarray
    predicted_active_count: int = 0


@dataclass
class ExecStats:
    predicted_sparsity: float = 0.0
    realized_sparsity: float = 0.0
    multiplies: int = 0
    pipeline: Pipeline = Pipeline.Dense
    predicted_active: int = 0
    revalidated: int = 0

    @staticmethod
    def from_c(s: capi.sg_exec_stats) -> "ExecStats":
        return ExecStats(s.predicted_sparsity, s.realized_sparsity, int(s.multiplies),
                         Pipeline(s.pipeline), int(s.predicted_active), int(s.revalidated))


@dataclass
class FfnResult:
    y: np.ndarray
    stats: ExecStats = field(default_factory=ExecStats)


@dataclass
class OpCounts:
    dense: int = 0
    sparse: float = 0.0
    ratio: float = 0.0


def validate_weights(w: FfnWeights) -> None:
    """types.hpp:31-51 (shape part; finiteness is checked by sg_layer_create)."""
    D, d = w.gate.shape
    if d < 1 or D < 1:
        raise DataError(f"ffn weights: gate must be at least 1x1, got {D}x{d}")
    if w.up.shape != (D, d):
        raise DataError(f"ffn weights: up is {w.up.shape[0]}x{w.up.shape[1]}, expected {D}x{d}")
    if w.down.shape != (d, D):
        raise DataError(
            f"ffn weights: down is {w.down.shape[0]}x{w.down.shape[1]}, expected {d}x{D}")


def validate_predictor(p: Predictor) -> None:
    """types.hpp:82-105 (shape part)."""
    if p.A.shape[1] != p.B.shape[0]:
        raise DataError(f"predictor: rank mismatch, A is {p.A.shape[0]}x{p.A.shape[1]} but B is "
                        f"{p.B.shape[0]}x{p.B.shape[1]}")
    if p.rank != p.A.shape[1]:
        raise DataError("predictor: rank field disagrees with factor shapes")
    if np.asarray(p.bias).shape != (p.A.shape[0],):
        raise DataError(f"predictor: bias length {np.asarray(p.bias).size} does not match "
                        f"intermediate size {p.A.shape[0]}")
    lim = min(p.A.shape[0], p.B.shape[1])
    if p.rank < 1 or p.rank > lim:
        raise DataError(f"predictor: rank {p.rank} out of range [1, {lim}]")


# ---------------------------------------------------------------------------
# device objects
# ---------------------------------------------------------------------------
class Context:
    """An sg_ctx: the per-stream device workspace (one per thread by default)."""

    def __init__(self, device: int = 0, max_hidden: int = 8192, max_inter: int = 32768,
                 max_rank: int = 8192):
        h = C.c_void_p()
        check(capi.lib().sg_ctx_create(device, max_hidden, max_inter, max_rank, C.byref(h)))
        self.handle = h
        self.device = device
        self.bounds = (max_hidden, max_inter, max_rank)

    def fits(self, d, D, r) -> bool:
        return d <= self.bounds[0] and D <= self.bounds[1] and r <= self.bounds[2]

    def close(self):
        if self.handle:
            capi.lib().sg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_context(device: int = 0, d: int = 1, D: int = 1, r: int = 1) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    ctx = ctxs.get(device)
    if ctx is None or not ctx.fits(d, D, r):
        b = (8192, 32768, 8192) if ctx is None else ctx.bounds
        ctx = Context(device, max(b[0], d), max(b[1], D), max(b[2], r))
        ctxs[device] = ctx
    return ctx


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class DeviceLayer:
    """An sg_layer: one FFN layer (or shard) resident in HBM as bf16.

    Built from reference-layout arrays (f64/f32, rounded f64->f32->bf16 RNE on
    upload) or from bf16 bit patterns (uint16) with ``down_neuron_major``.
    """

    def __init__(self, w: Optional[FfnWeights] = None, pred: Optional[Predictor] = None,
                 device: int = 0, shard_index: int = 0, shard_count: int = 1,
                 shard_interleave: bool = False, *, raw: Optional[dict] = None):
        desc = capi.sg_layer_desc()
        keep = []

        def ptr(a):
            keep.append(a)
            return a.ctypes.data_as(C.c_void_p)

        if raw is not None:
            # raw: dict(hidden, inter, rank, activation, gate, up, down_t, A, B (uint16), bias f32/f64)
            desc.hidden, desc.inter = raw["hidden"], raw["inter"]
            desc.rank = raw.get("rank", 0)
            desc.activation = int(raw.get("activation", 0))
            desc.weight_dtype = capi.SG_BF16
            desc.gate = ptr(np.ascontiguousarray(raw["gate"], dtype=np.uint16))
            desc.up = ptr(np.ascontiguousarray(raw["up"], dtype=np.uint16))
            desc.down = ptr(np.ascontiguousarray(raw["down_t"], dtype=np.uint16))
            desc.down_neuron_major = 1
            if raw.get("A") is not None:
                desc.pred_A = ptr(np.ascontiguousarray(raw["A"], dtype=np.uint16))
                desc.pred_B = ptr(np.ascontiguousarray(raw["B"], dtype=np.uint16))
                b = np.ascontiguousarray(raw["bias"])
                desc.bias_dtype = capi.SG_F32 if b.dtype == np.float32 else capi.SG_F64
                desc.bias = ptr(b.astype(np.float32 if b.dtype == np.float32 else np.float64))
            self.hidden, self.inter, self.rank = raw["hidden"], raw["inter"], desc.rank
        else:
            if w is None and pred is None:
                raise UsageError("DeviceLayer needs weights and/or a predictor")
            if w is not None:
                validate_weights(w)
                desc.hidden, desc.inter = w.hidden_size(), w.inter_size()
                desc.activation = int(w.activation)
                desc.gate, desc.up, desc.down = (ptr(_f64(w.gate)), ptr(_f64(w.up)),
                                                 ptr(_f64(w.down)))
            if pred is not None:
                validate_predictor(pred)
                if w is not None and pred.hidden_size() != w.hidden_size():
                    raise DataError("predictor input length does not match hidden size")
                if w is not None and pred.inter_size() != w.inter_size():
                    raise DataError("predictor intermediate size does not match weights")
                desc.hidden, desc.inter = pred.hidden_size(), pred.inter_size()
                desc.rank = int(pred.rank)
                desc.pred_A, desc.pred_B = ptr(_f64(pred.A)), ptr(_f64(pred.B))
                desc.bias_dtype = capi.SG_F64
                desc.bias = ptr(_f64(pred.bias))
            desc.weight_dtype = capi.SG_F64
            self.hidden, self.inter, self.rank = desc.hidden, desc.inter, desc.rank
        if raw is not None and raw.get("order") is not None:
            desc.neuron_order = ptr(np.ascontiguousarray(raw["order"], dtype=np.int64))
        desc.device = device
        desc.shard_index, desc.shard_count = shard_index, shard_count
        desc.shard_interleave = int(shard_interleave)
        h = C.c_void_p()
        check(capi.lib().sg_layer_create(C.byref(desc), C.byref(h)))
        self.handle = h
        self.device = device
        self.local_inter = int(capi.lib().sg_layer_local_inter(h))
        self.has_pred = desc.pred_A is not None

    def global_index(self, k: int) -> int:
        return int(capi.lib().sg_layer_global_index(self.handle, k))

    @property
    def device_bytes(self) -> int:
        return int(capi.lib().sg_layer_device_bytes(self.handle))

    def set_hot_rows(self, rows: int) -> None:
        """sg_layer_set_hot_rows: gate rows of the first `rows` neurons of every CTA block
        are fetched before the mask is known (0 = off). Timing only."""
        check(capi.lib().sg_layer_set_hot_rows(self.handle, int(rows)))

    def context(self) -> Context:
        return default_context(self.device, self.hidden, self.local_inter, max(self.rank, 1))

    def forward(self, x, pipeline: Pipeline = Pipeline.Sequential,
                ctx: Optional[Context] = None, stream: int = 0) -> FfnResult:
        """Host x (length d) -> FfnResult with host y (f64), through sg_ffn_forward."""
        ctx = ctx or self.context()
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
        y = np.zeros(self.hidden, dtype=np.float64)
        st = capi.sg_exec_stats()
        check(capi.lib().sg_ffn_forward(
            ctx.handle, self.handle, int(pipeline), x.ctypes.data_as(C.c_void_p), capi.SG_F64,
            x.size, y.ctypes.data_as(C.c_void_p), capi.SG_F64, C.byref(st), C.c_void_p(stream)))
        return FfnResult(y, ExecStats.from_c(st))

    def forward_device(self, x_ptr: int, y_ptr: int, pipeline: Pipeline,
                       ctx: Context, stream: int = 0) -> None:
        """Device fp32 x/y pointers, async on `stream` (no host sync)."""
        check(capi.lib().sg_ffn_forward_device(ctx.handle, self.handle, int(pipeline),
                                               C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                               C.c_void_p(stream)))

    def forward_batch(self, X, ctx: Optional[Context] = None, stream: int = 0):
        """Batched decode (sg_ffn_forward_batch_host): X (B, hidden) -> (Y (B, hidden) f64,
        per-token ExecStats, per-token predicted and survivor index arrays (global))."""
        ctx = ctx or self.context()
        X = np.ascontiguousarray(np.asarray(X, dtype=np.float32))
        if X.ndim != 2 or X.shape[1] != self.hidden:
            raise DataError("batch input must be (B, hidden)")
        B = X.shape[0]
        Y = np.zeros_like(X)
        st = (capi.sg_exec_stats * B)()
        check(capi.lib().sg_ffn_forward_batch_host(ctx.handle, self.handle,
                                                   X.ctypes.data_as(C.c_void_p), B,
                                                   Y.ctypes.data_as(C.c_void_p), st,
                                                   C.c_void_p(stream)))
        pb = np.zeros(self.local_inter, dtype=np.uint64)
        vb = np.zeros(self.local_inter, dtype=np.uint64)
        check(capi.lib().sg_ctx_read_batch(ctx.handle, C.c_void_p(stream), B, None,
                                           pb.ctypes.data_as(C.c_void_p),
                                           vb.ctypes.data_as(C.c_void_p)))
        gidx = np.array([self.global_index(k) for k in range(self.local_inter)], dtype=np.int64)
        P = [np.sort(gidx[((pb >> np.uint64(b)) & np.uint64(1)).astype(bool)]) for b in range(B)]
        V = [np.sort(gidx[((vb >> np.uint64(b)) & np.uint64(1)).astype(bool)]) for b in range(B)]
        return Y.astype(np.float64), [ExecStats.from_c(s) for s in st], P, V

    def forward_batch_residual(self, H, R, ctx: Optional[Context] = None, dense: bool = False):
        """Batched decode of a residual stream (sg_ffn_forward_batch_res): token b's input is
        H[b] + R[b] (e.g. h_{l+1} + y_l), summed in fp32 inside the launch. H, R: torch CUDA
        fp32 (B, hidden) tensors on this layer's device. Returns (Y torch tensor (B, hidden),
        per-token ExecStats)."""
        import torch
        ctx = ctx or self.context()
        if H.shape != R.shape or H.dim() != 2 or H.shape[1] != self.hidden:
            raise DataError("batch input must be (B, hidden) and match the residual")
        H = H.contiguous().float()
        R = R.contiguous().float()
        Y = torch.zeros_like(H)
        B = H.shape[0]
        sh = torch.cuda.current_stream(self.device).cuda_stream
        check(capi.lib().sg_ffn_forward_batch_res(ctx.handle, self.handle, C.c_void_p(H.data_ptr()),
                                                  C.c_void_p(R.data_ptr()), B, C.c_void_p(Y.data_ptr()),
                                                  1 if dense else 0, None, None, C.c_void_p(sh)))
        st = (capi.sg_exec_stats * B)()
        check(capi.lib().sg_ctx_read_batch(ctx.handle, C.c_void_p(sh), B, st, None, None))
        return Y, [ExecStats.from_c(x) for x in st]

    def forward_batch_dense(self, X, ctx: Optional[Context] = None) -> np.ndarray:
        """Dense batched comparator (sg_ffn_forward_batch_dense): dense_ffn for every token
        of X (B, hidden), every row read once on the tensor cores. Returns Y (B, hidden)."""
        import torch
        ctx = ctx or self.context()
        X = np.ascontiguousarray(np.asarray(X, dtype=np.float32))
        xt = torch.tensor(X, device=f"cuda:{self.device}")
        yt = torch.zeros_like(xt)
        sh = torch.cuda.current_stream(self.device).cuda_stream
        check(capi.lib().sg_ffn_forward_batch_dense(ctx.handle, self.handle, C.c_void_p(xt.data_ptr()),
                                                    X.shape[0], C.c_void_p(yt.data_ptr()),
                                                    C.c_void_p(sh)))
        check(capi.lib().sg_ctx_read_batch(ctx.handle, C.c_void_p(sh), X.shape[0], None, None, None))
        return yt.double().cpu().numpy()

    def predict_mask(self, x, ctx: Optional[Context] = None, stream: int = 0) -> Mask:
        ctx = ctx or self.context()
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
        mask = np.zeros(self.local_inter, dtype=np.uint8)
        cnt = C.c_int64(0)
        check(capi.lib().sg_predict_mask(ctx.handle, self.handle, x.ctypes.data_as(C.c_void_p),
                                         capi.SG_F64, x.size, mask.ctypes.data_as(C.c_void_p),
                                         C.byref(cnt), C.c_void_p(stream)))
        return Mask(mask, int(cnt.value))

    def close(self):
        if getattr(self, "handle", None):
            capi.lib().sg_layer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_stats(ctx: Context, stream: int = 0) -> ExecStats:
    st = capi.sg_exec_stats()
    check(capi.lib().sg_ctx_read_stats(ctx.handle, C.c_void_p(stream), C.byref(st)))
    return ExecStats.from_c(st)


def read_sets(ctx: Context, capacity: int, stream: int = 0):
    """(P, V, g over P, z over V) of the ctx's last sparse call, global indices."""
    P = np.zeros(capacity, dtype=np.int32)
    V = np.zeros(capacity, dtype=np.int32)
    g = np.zeros(capacity, dtype=np.float32)
    z = np.zeros(capacity, dtype=np.float32)
    p, v = C.c_int64(0), C.c_int64(0)
    check(capi.lib().sg_ctx_read_sets(ctx.handle, C.c_void_p(stream),
                                      P.ctypes.data_as(C.c_void_p), C.byref(p),
                                      V.ctypes.data_as(C.c_void_p), C.byref(v),
                                      g.ctypes.data_as(C.c_void_p), z.ctypes.data_as(C.c_void_p)))
    return P[:p.value], V[:v.value], g[:p.value], z[:v.value]


# ---------------------------------------------------------------------------
# stateless reference API
# ---------------------------------------------------------------------------
_cache: dict = {}
_cache_lock = threading.Lock()


def _fingerprint(*arrays) -> bytes:
    """Digest of the FULL contents of the arrays: any in-place change of weights
    (or a swapped array) gives a new device layer — which re-runs the upload
    validation, so a NaN written into cached weights still raises DataError as
    the reference's per-call validate does (types.hpp:31-51, ffn_exec.hpp:57).
    blake2b runs at ~1 GB/s, well under the upload's own cost."""
    h = hashlib.blake2b(digest_size=16)
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(repr((a.dtype.str, a.shape)).encode())
        h.update(memoryview(a).cast("B"))
    return h.digest()


def _layer_for(w: Optional[FfnWeights], pred: Optional[Predictor], device: int = 0) -> DeviceLayer:
    fp = _fingerprint(*(() if w is None else (w.gate, w.up, w.down)),
                      *(() if pred is None else (pred.A, pred.B, pred.bias)))
    key = (id(w), id(pred), device, fp, None if w is None else int(w.activation),
           None if pred is None else int(pred.rank))
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None:
            wref, pref, layer = hit
            if (w is None or wref() is w) and (pred is None or pref() is pred):
                return layer
    layer = DeviceLayer(w, pred, device)
    with _cache_lock:
        for k in [k for k in _cache if k[:3] == key[:3]]:  # superseded contents of the same objects
            _cache.pop(k, None)
        _cache[key] = (weakref.ref(w) if w is not None else (lambda: None),
                       weakref.ref(pred) if pred is not None else (lambda: None), layer)
        for obj in (w, pred):
            if obj is not None:
                weakref.finalize(obj, _cache.pop, key, None)
    return layer


def dense_ffn(w: FfnWeights, x) -> FfnResult:
    """ffn_exec.hpp:103-122 on the GPU (dense gather-free GEMV FFN)."""
    return _layer_for(w, None).forward(x, Pipeline.Dense)


def predict_mask(pred: Predictor, x) -> Mask:
    """ffn_exec.hpp:125-146 on the GPU (stage 1)."""
    validate_predictor(pred)
    return _layer_for(None, pred).predict_mask(x)


def sparse_ffn_parallel(w: FfnWeights, pred: Predictor, x) -> FfnResult:
    """ffn_exec.hpp:149-178 on the GPU."""
    return _layer_for(w, pred).forward(x, Pipeline.Parallel)


def sparse_ffn_sequential(w: FfnWeights, pred: Predictor, x) -> FfnResult:
    """ffn_exec.hpp:183-218 on the GPU (the five-stage hot path)."""
    return _layer_for(w, pred).forward(x, Pipeline.Sequential)


def op_count_model(d: int, D: int, r: int, s: float, s_prime: float) -> OpCounts:
    """ffn_exec.hpp:229-244 (host arithmetic in the C library)."""
    dense, sparse, ratio = C.c_int64(0), C.c_double(0), C.c_double(0)
    check(capi.lib().sg_op_count_model(d, D, r, s, s_prime, C.byref(dense), C.byref(sparse),
                                       C.byref(ratio)))
    return OpCounts(dense.value, sparse.value, ratio.value)


def round_bf16(a) -> np.ndarray:
    """The upload rounding (f64 -> f32 -> bf16, RNE) as uint16 bit patterns."""
    a = _f64(a)
    out = np.zeros(a.shape, dtype=np.uint16)
    capi.lib().sg_round_bf16(a.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p), a.size)
    return out


def bf16_to_f64(bits) -> np.ndarray:
    bits = np.asarray(bits, dtype=np.uint16)
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
