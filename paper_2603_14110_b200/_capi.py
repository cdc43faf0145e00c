"""ctypes binding of the C ABI in include/sparsegate_c.h (libsparsegate_b200.so).

This is the only way Python reaches the executor: every call goes through the
same extern "C" entry points a C/C++ caller (include/sparsegate/ffn_exec.hpp)
uses. There is no CPU fallback: if the shared library is missing the import
raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SG_LIB=timing selects the instrumented build (per-phase %globaltimer stamps,
# tools/phase_profile.py); the default is the production library.
LIB_PATH = os.path.join(HERE, f"libsparsegate_b200_{os.environ['SG_LIB']}.so" if os.environ.get("SG_LIB")
                        else "libsparsegate_b200.so")

SG_OK, SG_ERR_USAGE, SG_ERR_DATA, SG_ERR_PROPERTY, SG_ERR_IO, SG_ERR_CUDA, SG_ERR_NCCL = range(7)
SG_F64, SG_F32, SG_BF16 = 0, 1, 2
SG_PIPELINE_DENSE, SG_PIPELINE_PARALLEL, SG_PIPELINE_SEQUENTIAL = 0, 1, 2


class sg_exec_stats(C.Structure):
    _fields_ = [
        ("predicted_sparsity", C.c_double),
        ("realized_sparsity", C.c_double),
        ("multiplies", C.c_int64),
        ("pipeline", C.c_int32),
        ("pad_", C.c_int32),
        ("predicted_active", C.c_int64),
        ("revalidated", C.c_int64),
    ]


class sg_layer_desc(C.Structure):
    _fields_ = [
        ("hidden", C.c_int64),
        ("inter", C.c_int64),
        ("rank", C.c_int64),
        ("activation", C.c_int32),
        ("weight_dtype", C.c_int32),
        ("bias_dtype", C.c_int32),
        ("device", C.c_int32),
        ("gate", C.c_void_p),
        ("up", C.c_void_p),
        ("down", C.c_void_p),
        ("pred_A", C.c_void_p),
        ("pred_B", C.c_void_p),
        ("bias", C.c_void_p),
        ("shard_index", C.c_int32),
        ("shard_count", C.c_int32),
        ("shard_interleave", C.c_int32),
        ("down_neuron_major", C.c_int32),
        ("neuron_order", C.c_void_p),
    ]


# (name, restype, argtypes) for every symbol declared in include/sparsegate_c.h
_VP, _I32, _I64, _D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
SYMBOLS = [
    ("sg_last_error", C.c_char_p, []),
    ("sg_version", C.c_char_p, []),
    ("sg_layer_create", C.c_int, [C.POINTER(sg_layer_desc), C.POINTER(_VP)]),
    ("sg_layer_destroy", C.c_int, [_VP]),
    ("sg_layer_local_inter", _I64, [_VP]),
    ("sg_layer_global_index", _I64, [_VP, _I64]),
    ("sg_layer_device_bytes", _I64, [_VP]),
    ("sg_layer_set_hot_rows", C.c_int, [_VP, _I64]),
    ("sg_ctx_create", C.c_int, [_I32, _I64, _I64, _I64, C.POINTER(_VP)]),
    ("sg_ctx_destroy", C.c_int, [_VP]),
    ("sg_ffn_forward_device", C.c_int, [_VP, _VP, C.c_int, _VP, _VP, _VP]),
    ("sg_ctx_read_stats", C.c_int, [_VP, _VP, C.POINTER(sg_exec_stats)]),
    ("sg_ctx_read_sets", C.c_int, [_VP, _VP, _VP, C.POINTER(_I64), _VP, C.POINTER(_I64), _VP, _VP]),
    ("sg_predict_mask", C.c_int, [_VP, _VP, _VP, C.c_int, _I64, _VP, C.POINTER(_I64), _VP]),
    ("sg_ffn_forward", C.c_int, [_VP, _VP, C.c_int, _VP, C.c_int, _I64, _VP, C.c_int,
                                 C.POINTER(sg_exec_stats), _VP]),
    ("sg_ffn_forward_layers", C.c_int, [_VP, _VP, _I32, C.c_int, _VP, _VP, _I32, _VP]),
    ("sg_ffn_forward_layers_host", C.c_int, [_VP, _VP, _I32, C.c_int, _VP, _VP, _I32,
                                             C.POINTER(sg_exec_stats), _VP]),
    ("sg_ctx_read_stack_stats", C.c_int, [_VP, _VP, _I32, C.POINTER(sg_exec_stats)]),
    ("sg_ctx_enable_stack_sets", C.c_int, [_VP, _I32]),
    ("sg_ctx_read_stack_sets", C.c_int, [_VP, _VP, _I32, _VP, C.POINTER(_I64), _VP, C.POINTER(_I64)]),
    ("sg_ffn_forward_batch", C.c_int, [_VP, _VP, _VP, _I32, _VP, _VP]),
    ("sg_ctx_enable_tc_trace", C.c_int, [_VP, _I32]),
    ("sg_ctx_read_tc_trace", C.c_int, [_VP, _VP, _I32, _VP, C.POINTER(_I32)]),
    ("sg_tc_unit_codes", C.c_int, [_VP, _VP, _I32]),
    ("sg_ffn_forward_batch_dense", C.c_int, [_VP, _VP, _VP, _I32, _VP, _VP]),
    ("sg_ffn_forward_batch_res", C.c_int, [_VP, _VP, _VP, _VP, _I32, _VP, _I32, _VP, _VP, _VP]),
    ("sg_ctx_read_batch", C.c_int, [_VP, _VP, _I32, C.POINTER(sg_exec_stats), _VP, _VP]),
    ("sg_ffn_forward_batch_host", C.c_int, [_VP, _VP, _VP, _I32, _VP, C.POINTER(sg_exec_stats), _VP]),
    ("sg_ctx_enable_phase_timing", C.c_int, [_VP, _I32]),
    ("sg_ctx_read_phase_timing", C.c_int, [_VP, _VP, _I32, _VP, C.POINTER(_I32)]),
    ("sg_comm_unique_id", C.c_int, [_VP]),
    ("sg_comm_create", C.c_int, [_I32, _I32, _I32, _VP, C.POINTER(_VP)]),
    ("sg_comm_destroy", C.c_int, [_VP]),
    ("sg_comm_size", _I32, [_VP]),
    ("sg_comm_rank", _I32, [_VP]),
    ("sg_allreduce_sum", C.c_int, [_VP, _VP, _I64, _VP]),
    ("sg_ffn_forward_layers_sharded", C.c_int, [_VP, _VP, _VP, _I32, C.c_int, _VP, _VP, _I32, _VP]),
    ("sg_layer_hidden", _I64, [_VP]),
    ("sg_op_count_model", C.c_int, [_I64, _I64, _I64, _D, _D, C.POINTER(_I64), C.POINTER(_D),
                                    C.POINTER(_D)]),
    ("sg_round_bf16", None, [_VP, _VP, _I64]),
    ("sg_shard_range", C.c_int, [_I64, _I32, _I32, _I32, C.POINTER(_I64), C.POINTER(_I64),
                                 C.POINTER(_I64)]),
    ("sg_exec_stats_from_counts", C.c_int, [_I64, _I64, _I64, C.c_int, _I64, _I64,
                                            C.POINTER(sg_exec_stats)]),
    ("sg_synthetic_fixture", C.c_int, [_I64, _I64, _I64, _I64, _D, C.c_uint64, _VP, _VP, _VP,
                                       _VP, _VP]),
    ("sg_synthetic_fixture_bf16", C.c_int, [_I64, _I64, _I64, _I64, _D, C.c_uint64, _VP, _VP,
                                            _VP, _VP, _VP]),
    ("sg_predict_mask_f64", C.c_int, [_I32, _VP, _VP, _VP, _I64, _I64, _I64, _VP, _VP, C.POINTER(_I64)]),
    ("sg_cholesky_whitening", C.c_int, [_VP, _I64, _I64, _D, _VP, _I32, _VP, _VP, C.POINTER(_D)]),
    ("sg_build_predictor", C.c_int, [_VP, _I64, _I64, _VP, _I64, _I64, _I32, _I32, C.c_uint64, _D, _VP,
                                     _I32, _VP, _VP, _VP, _I64, C.POINTER(_D), C.POINTER(_D)]),
    ("sg_singular_values", C.c_int, [_VP, _I64, _I64, _I32, _I64, C.c_uint64, _VP]),
    ("sg_proxy_scores", C.c_int, [_VP, _VP, _I64, _I64, _I64, _VP, _I64, _VP]),
    ("sg_damage_weights", C.c_int, [_VP, _VP, _VP, _I64, _I64, _I32, _VP, _I64, _VP]),
    ("sg_greedy_calibrate", C.c_int, [_VP, _VP, _I64, _I64, _I32, _D, _VP, C.POINTER(_D),
                                      C.POINTER(_D)]),
]

_lib = None


def lib():
    """Load libsparsegate_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_2603_14110_b200/csrc). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SYMBOLS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
