"""The d_ff-sharded decode step behind the C ABI (sg_comm_*, sg_ffn_forward_layers_sharded;
SURVEY.md §8e): per-layer launches on the rank's shard + one NCCL all-reduce per layer,
issued from C++ (csrc/sg_comm.cpp).

One GPU per gpurun call: a single-rank communicator exercises the whole C++ path
(NCCL init through dlopen, the per-layer launch with residual input, the in-place
all-reduce, graph capture) and must reproduce the one-launch stack bit for bit. The
multi-rank exchange itself is covered on CPU (tests/test_sharded_cpu.py, gloo), and
shards run one after the other must sum to the full layer (test_gpu_scale.py).
"""
import ctypes as C

import numpy as np
import pytest

from paper_2603_14110_b200 import DeviceLayer, Pipeline
from paper_2603_14110_b200 import _capi as capi
from paper_2603_14110_b200.ffn_exec import Context, check
from test_gpu_parity import _calibrated_layer

pytestmark = pytest.mark.gpu


def _comm1():
    lib = capi.lib()
    uid = (C.c_uint8 * 128)()
    check(lib.sg_comm_unique_id(uid))
    h = C.c_void_p()
    check(lib.sg_comm_create(0, 1, 0, uid, C.byref(h)))
    assert lib.sg_comm_size(h) == 1 and lib.sg_comm_rank(h) == 0
    return h


@pytest.mark.parametrize("chain", [0, 1, 2])
def test_sharded_step_single_rank_equals_stack(chain):
    import torch
    lib = capi.lib()
    d, D, r = 512, 1408, 64
    layers, xs = [], []
    for s in range(3):
        fx, pred = _calibrated_layer(d, D, r, seed=300 + s)
        layers.append(DeviceLayer(fx.weights, pred))
        xs.append(fx.eval[:, 0])
    arr = (C.c_void_p * 3)(*[l.handle.value for l in layers])
    xt = torch.tensor(np.stack(xs), dtype=torch.float32, device="cuda")
    ctx = Context(0, d, D, r)
    sh = torch.cuda.current_stream().cuda_stream
    y_stack = torch.zeros_like(xt)
    check(lib.sg_ffn_forward_layers(ctx.handle, arr, 3, int(Pipeline.Sequential), C.c_void_p(xt.data_ptr()),
                                    C.c_void_p(y_stack.data_ptr()), chain, C.c_void_p(sh)))
    st_stack = (capi.sg_exec_stats * 3)()
    check(lib.sg_ctx_read_stack_stats(ctx.handle, C.c_void_p(sh), 3, st_stack))
    comm = _comm1()
    try:
        y_sh = torch.zeros_like(xt)
        check(lib.sg_ffn_forward_layers_sharded(ctx.handle, comm, arr, 3, int(Pipeline.Sequential),
                                                C.c_void_p(xt.data_ptr()), C.c_void_p(y_sh.data_ptr()),
                                                chain, C.c_void_p(sh)))
        st_sh = (capi.sg_exec_stats * 3)()
        check(lib.sg_ctx_read_stack_stats(ctx.handle, C.c_void_p(sh), 3, st_sh))
        assert torch.equal(y_sh, y_stack)
        assert [(s.predicted_active, s.revalidated) for s in st_sh] == \
               [(s.predicted_active, s.revalidated) for s in st_stack]
        # the whole step (3 launches + 3 all-reduces) captured in one CUDA graph
        cs = torch.cuda.Stream()
        y_g = torch.zeros_like(xt)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            check(lib.sg_ffn_forward_layers_sharded(ctx.handle, comm, arr, 3, int(Pipeline.Sequential),
                                                    C.c_void_p(xt.data_ptr()), C.c_void_p(y_g.data_ptr()),
                                                    chain, C.c_void_p(cs.cuda_stream)))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y_g, y_stack)
    finally:
        lib.sg_comm_destroy(comm)


def test_allreduce_single_rank_identity_and_errors():
    import torch
    lib = capi.lib()
    comm = _comm1()
    try:
        v = torch.arange(1000, dtype=torch.float32, device="cuda")
        w = v.clone()
        check(lib.sg_allreduce_sum(comm, C.c_void_p(w.data_ptr()), 1000,
                                   C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        assert torch.equal(v, w)
        assert lib.sg_ffn_forward_layers_sharded(None, comm, None, 0, 2, None, None, 0, None) != 0
        assert lib.sg_ffn_forward_layers_sharded(None, None, None, 0, 2, None, None, 0, None) != 0
    finally:
        lib.sg_comm_destroy(comm)
