"""Multi-GPU decode: the FFN intermediate dimension sharded over ranks.

One process per GPU. Rank k holds neurons shard_range(inter, k, N) of every layer
(gate/up rows, down columns, predictor A rows and bias entries) and the full
predictor factor B. A token's layer is then

    t = B x                        (every rank, redundant: r*d MACs, r*d*2 bytes)
    partial_k = sum_{i in shard k} z_i down_i      (the sm_100a executor, local)
    y = sum_k partial_k            (ONE all-reduce of d fp32 per layer)

The sets P and V are unions of disjoint per-shard sets, so |P| and |V| are sums
and the layer's ExecStats follow from the summed counts with the reference
formulas (ffn_exec.hpp:173-180, :209-216) over the global inter; the only
exchange is the d-vector sum (plus two int64 counts when stats are requested).

The exchange code below is backend-agnostic: NCCL on device tensors in
production, gloo on host tensors in the CPU tests (tests/test_sharded_cpu.py).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import numpy as np

from . import _capi as capi
from .ffn_exec import (Context, DeviceLayer, ExecStats, FfnResult, FfnWeights, Pipeline,
                       Predictor, check, read_stats)


def shard_range(inter: int, index: int, count: int, interleave: bool = False) -> Tuple[int, int, int]:
    """(base, stride, count): the global neurons base + k*stride a shard holds."""
    b, s, n = C.c_int64(), C.c_int64(), C.c_int64()
    check(capi.lib().sg_shard_range(inter, index, count, int(interleave), C.byref(b), C.byref(s),
                                    C.byref(n)))
    return int(b.value), int(s.value), int(n.value)


def shard_indices(inter: int, index: int, count: int, interleave: bool = False) -> np.ndarray:
    base, stride, n = shard_range(inter, index, count, interleave)
    return base + stride * np.arange(n, dtype=np.int64)


def stats_from_counts(hidden: int, inter: int, rank: int, pipeline: Pipeline, p: int,
                      v: int) -> ExecStats:
    """Whole-layer ExecStats from |P|, |V| summed over shards (sg_exec_stats_from_counts)."""
    st = capi.sg_exec_stats()
    check(capi.lib().sg_exec_stats_from_counts(hidden, inter, rank, int(pipeline), int(p), int(v),
                                               C.byref(st)))
    return ExecStats.from_c(st)


def combine_shards(y_partial, p: int, v: int, hidden: int, inter: int, rank: int,
                   pipeline: Pipeline, group=None, with_stats: bool = True):
    """Sum the per-shard outputs in place (one all-reduce) and, optionally, the
    (|P|, |V|) counts (a second, 16-byte all-reduce); returns the layer's ExecStats.

    y_partial: torch tensor on the backend's device (cuda for NCCL, cpu for gloo).
    """
    import torch
    import torch.distributed as dist

    dist.all_reduce(y_partial, group=group)
    if not with_stats:
        return None
    cnt = torch.tensor([p, v], dtype=torch.int64, device=y_partial.device)
    dist.all_reduce(cnt, group=group)
    P, V = (int(a) for a in cnt.tolist())
    return stats_from_counts(hidden, inter, rank, pipeline, P, V)


class ShardedLayer:
    """This rank's shard of one layer, plus the exchange that completes it.

    `weights`/`predictor` describe the FULL layer (reference layouts); only this
    rank's neurons are uploaded. Requires torch.distributed to be initialised
    (NCCL for cuda tensors).
    """

    def __init__(self, weights: Optional[FfnWeights], predictor: Optional[Predictor],
                 device: int, group=None, interleave: bool = False, *, raw: Optional[dict] = None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.index = dist.get_rank(group)
        self.layer = DeviceLayer(weights, predictor, device, shard_index=self.index,
                                 shard_count=self.world, shard_interleave=interleave, raw=raw)
        self.hidden, self.inter, self.rank = self.layer.hidden, self.layer.inter, self.layer.rank

    def forward_device(self, x, y, pipeline: Pipeline, ctx: Context, stream: int = 0) -> None:
        """x, y: cuda fp32 tensors of length hidden. y = full layer output after return
        (stream-ordered; NCCL runs on the current torch stream, which must be `stream`)."""
        self.layer.forward_device(x.data_ptr(), y.data_ptr(), pipeline, ctx, stream)
        combine_shards(y, 0, 0, self.hidden, self.inter, self.rank, pipeline, self.group,
                       with_stats=False)

    def forward(self, x, pipeline: Pipeline = Pipeline.Sequential,
                ctx: Optional[Context] = None) -> FfnResult:
        """Host x -> FfnResult (host y f64, whole-layer stats): the reference call shape."""
        import torch

        ctx = ctx or self.layer.context()
        dev = torch.device("cuda", self.layer.device)
        stream = torch.cuda.current_stream(dev).cuda_stream
        xt = torch.as_tensor(np.asarray(x, dtype=np.float32).reshape(-1)).to(dev)
        if xt.numel() != self.hidden or not bool(torch.isfinite(xt).all()):
            from .ffn_exec import DataError
            raise DataError("input length mismatch or non-finite input")
        yt = torch.empty(self.hidden, dtype=torch.float32, device=dev)
        self.layer.forward_device(xt.data_ptr(), yt.data_ptr(), pipeline, ctx, stream)
        local = read_stats(ctx, stream)
        st = combine_shards(yt, local.predicted_active, local.revalidated, self.hidden,
                            self.inter, self.rank, pipeline, self.group)
        return FfnResult(yt.double().cpu().numpy(), st)
