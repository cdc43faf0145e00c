"""CPU: the calibration-balanced neuron layout (model.balanced_order) that the
bench uploads with sg_layer_desc.neuron_order and sg_layer_set_hot_rows."""
import numpy as np

from paper_2603_14110_b200.model import balanced_order


def _blocks(order, G):
    n = len(order)
    bounds = [c * n // G for c in range(G + 1)]  # the kernel's split (split_lo)
    return [order[bounds[c]:bounds[c + 1]] for c in range(G)]


def test_balanced_order_is_a_permutation_with_kernel_block_sizes():
    rng = np.random.default_rng(0)
    D, G = 11008, 148
    load = rng.gamma(0.5, 1.0, D)
    order = balanced_order(load, np.arange(D, dtype=np.int64), G)
    assert sorted(order.tolist()) == list(range(D))
    sizes = [len(b) for b in _blocks(order, G)]
    assert max(sizes) - min(sizes) <= 1


def test_balanced_order_balances_expected_load_and_puts_hot_first():
    rng = np.random.default_rng(1)
    D, G = 4096, 64
    load = rng.gamma(0.5, 1.0, D)
    order = balanced_order(load, np.arange(D, dtype=np.int64), G)
    blocks = _blocks(order, G)
    per = np.array([load[b].sum() for b in blocks])
    naive = np.array([load[b].sum() for b in _blocks(np.arange(D), G)])
    assert per.max() / per.mean() < naive.max() / naive.mean()
    assert per.max() / per.mean() < 1.15
    for b in blocks:  # each block leads with its most loaded neurons (the hot prefix)
        assert np.all(np.diff(load[b]) <= 0)


def test_balanced_order_of_a_shard_subset():
    rng = np.random.default_rng(2)
    D, G = 3000, 37
    load = rng.random(D)
    mine = np.arange(1, D, 2, dtype=np.int64)  # interleaved shard
    order = balanced_order(load, mine, G)
    assert sorted(order.tolist()) == mine.tolist()
