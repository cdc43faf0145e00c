"""CPU: the multi-GPU (d_ff-sharded) host logic, SURVEY.md §8e.

The shard map and the whole-layer stats come from the product library
(sg_shard_range / sg_exec_stats_from_counts, pure host); the exchange is
paper_2603_14110_b200.sharded.combine_shards run over gloo with world_size 2.
Per-shard compute is played by the f64 oracle restricted to the shard's
neurons (the test is the checker; the exchange and the stats are under test).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2603_14110_b200 import Pipeline
from paper_2603_14110_b200.sharded import (combine_shards, shard_indices, shard_range,
                                           stats_from_counts)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("inter", [1, 7, 256, 11008, 14336])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("interleave", [False, True])
def test_shards_partition_the_layer(inter, world, interleave):
    idx = [shard_indices(inter, k, world, interleave) for k in range(world)]
    allidx = np.sort(np.concatenate(idx))
    assert np.array_equal(allidx, np.arange(inter))
    sizes = [len(i) for i in idx]
    assert max(sizes) - min(sizes) <= 1
    for i in idx:
        assert np.all(np.diff(i) > 0)


def test_shard_range_errors():
    from paper_2603_14110_b200 import UsageError, DataError
    with pytest.raises(UsageError):
        shard_range(100, 2, 2)
    with pytest.raises(UsageError):
        shard_range(100, -1, 2)
    with pytest.raises(DataError):
        shard_range(0, 0, 1)
    assert shard_range(100, 0, 0) == (0, 1, 100)  # shard_count 0 = unsharded


def test_stats_from_counts_matches_reference_formulas():
    d, D, r = 4096, 11008, 256
    for pipe in (Pipeline.Dense, Pipeline.Parallel, Pipeline.Sequential):
        st = stats_from_counts(d, D, r, pipe, 5504, 1100)
        if pipe == Pipeline.Dense:
            assert st.multiplies == 3 * d * D and st.predicted_sparsity == 0.0
        elif pipe == Pipeline.Parallel:
            assert st.multiplies == r * (d + D) + 3 * d * 5504
            assert st.predicted_sparsity == 1.0 - 5504 / D == st.realized_sparsity
        else:
            assert st.multiplies == r * (d + D) + d * 5504 + 2 * d * 1100
            assert st.realized_sparsity == 1.0 - 1100 / D
    from paper_2603_14110_b200 import UsageError
    with pytest.raises(UsageError):
        stats_from_counts(d, D, r, Pipeline.Sequential, 10, 11)  # |V| > |P|


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, interleave, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        g = dict(np.load(os.path.join(GOLD, "synthetic_exec_h64_i256_r16.npz")))
        d, D = g["gate"].shape[1], g["gate"].shape[0]
        r = g["B"].shape[0]
        idx = shard_indices(D, rank, world, interleave)
        out = []
        for act in (0, 1):
            for pipe in (Pipeline.Parallel, Pipeline.Sequential):
                for x in g["xs"][:4]:
                    o = O.sparse_ffn(g["gate"][idx], g["up"][idx], g["down"][:, idx], g["A"][idx],
                                     g["B"], g["bias"][idx], x, act, int(pipe))
                    y = torch.tensor(o.y, dtype=torch.float64)
                    st = combine_shards(y, len(o.P), len(o.V), d, D, r, pipe)
                    Pg = idx[o.P]
                    allP = [None] * world
                    dist.all_gather_object(allP, Pg.tolist())
                    out.append((y.numpy(), st, sorted(sum(allP, []))))
        q.put((rank, out, None))
        dist.destroy_process_group()
    except Exception as e:  # surface failures to the parent
        q.put((rank, None, repr(e)))


@pytest.mark.parametrize("interleave", [False, True])
def test_two_rank_gloo_exchange_matches_unsharded_oracle(interleave):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, interleave, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, out, err = q.get(timeout=240)
        assert err is None, err
        res[rank] = out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = dict(np.load(os.path.join(GOLD, "synthetic_exec_h64_i256_r16.npz")))
    k = 0
    for act in (0, 1):
        for pipe in (1, 2):
            for x in g["xs"][:4]:
                full = O.sparse_ffn(g["gate"], g["up"], g["down"], g["A"], g["B"], g["bias"], x,
                                    act, pipe)
                for rank in range(world):
                    y, st, P = res[rank][k]
                    # the all-reduce re-associates the f64 sum across 2 shards
                    assert np.allclose(y, full.y, rtol=1e-12, atol=1e-12 * np.abs(full.y).max())
                    assert st.multiplies == full.stats.multiplies
                    assert st.predicted_sparsity == full.stats.predicted_sparsity
                    assert st.realized_sparsity == full.stats.realized_sparsity
                    assert P == full.P.tolist()
                assert np.array_equal(res[0][k][0], res[1][k][0])  # ranks agree bitwise
                k += 1
