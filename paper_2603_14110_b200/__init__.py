"""sparsegate-b200: B200-native sparse gated-FFN decode executor.

A from-scratch sm_100a implementation of the decode hot path of "SVD
Contextual Sparsity Predictors for Fast LLM Inference" (arXiv 2603.14110),
behind the reference executor API (proj/include/sparsegate/ffn_exec.hpp).

Layout:
  csrc/sg_kernels.cu   persistent cooperative executor kernels (sm_100a)
  csrc/sg_host.cpp     C ABI (include/sparsegate_c.h): upload, validation, stats
  _capi.py             ctypes binding of that ABI
  ffn_exec.py          the reference API mirror (dense_ffn, predict_mask, ...)
  synthetic.py         synthetic.hpp fixtures (bit-identical stream)
  offline.py           host-side predictor build + greedy calibration
"""
from .ffn_exec import (  # noqa: F401
    Activation, Context, CudaError, DataError, DeviceLayer, Error, ExecStats, FfnResult,
    FfnWeights, IoError, Mask, OpCounts, Pipeline, Predictor, PropertyViolation, UsageError,
    bf16_to_f64, dense_ffn, op_count_model, predict_mask, read_sets, read_stats, round_bf16,
    sparse_ffn_parallel, sparse_ffn_sequential,
)
