"""CPU: the C-ABI library (libsparsegate_b200.so) loads, exports every symbol
include/sparsegate_c.h declares, and its pure-host entry points match the
reference (no device compute here — there is no GPU in this container)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2603_14110_b200 import _capi as capi
from paper_2603_14110_b200 import op_count_model, round_bf16
from paper_2603_14110_b200.ffn_exec import DataError, UsageError
from paper_2603_14110_b200.offline import greedy_calibrate
from paper_2603_14110_b200.synthetic import SyntheticConfig, make_synthetic_fixture

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "sparsegate_c.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(sg_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(capi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 26
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes table binds exactly the header's functions
    assert sorted(n for n, _, _ in capi.SYMBOLS) == syms


def test_version_and_error_channel():
    lib = capi.lib()
    assert lib.sg_version().decode().startswith("sparsegate-b200")
    st = lib.sg_layer_create(None, None)
    assert st == capi.SG_ERR_USAGE
    assert lib.sg_last_error().decode() != ""


def test_op_count_model_matches_reference_kat():
    """ffn_exec_tests.cpp:256-279."""
    oc = op_count_model(4096, 11008, 256, 0.5, 0.9)
    assert oc.dense == 135266304
    assert abs(oc.sparse - 35428761.6) < 1e-6
    assert f"{oc.ratio:.2f}" == "3.82"
    rows = np.load(os.path.join(GOLD, "op_count.npz"))["rows"]
    for d, D, r, s, sp, dense, sparse, ratio in rows:
        got = op_count_model(int(d), int(D), int(r), s, sp)
        assert (got.dense, got.sparse, got.ratio) == (int(dense), sparse, ratio)
    with pytest.raises(DataError):
        op_count_model(64, 256, 8, 0.9, 0.5)  # s' < s
    with pytest.raises(DataError):
        op_count_model(0, 256, 8, 0.5, 0.9)


def test_round_bf16_is_rne_through_f32():
    import torch
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(4096) * 10.0 ** rng.integers(-30, 30, 4096),
                        [0.0, -0.0, np.inf, -np.inf, 1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8,
                         3.3895313892515355e38, 1e-45, -1e-40]])
    got = round_bf16(x)
    want = torch.tensor(x.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy()
    assert np.array_equal(got.view(np.int16), want)
    nan = round_bf16(np.array([np.nan]))
    assert (int(nan[0]) & 0x7F80) == 0x7F80 and (int(nan[0]) & 0x7F) != 0


def test_synthetic_fixture_matches_reference_stream():
    """synthetic.hpp:80-108: product generator == reference generator bit-for-bit."""
    g = np.load(os.path.join(GOLD, "synthetic_h32_i128_s9.npz"))
    f = make_synthetic_fixture(SyntheticConfig(32, 128, 128, 32, natural_sparsity=0.9, seed=9))
    got = {"gate": f.weights.gate, "up": f.weights.up, "down": f.weights.down, "calib": f.calib,
           "eval": f.eval}
    for k in got:
        assert np.array_equal(got[k], g[k]), k
    with pytest.raises(DataError):
        make_synthetic_fixture(SyntheticConfig(32, 128, 128, 32, natural_sparsity=1.0, seed=9))


def _calib(scores, weights, eta, target):
    return greedy_calibrate(np.array(scores, float), np.array(weights, float), eta, target)


def test_greedy_calibration_reference_kats():
    """calibration_tests.cpp:150-228."""
    S, W = [[1, 2, 3, 4], [1, 2, 3, 4]], [[0, 1, 2, 3], [0, 0, 5, 6]]
    r = _calib(S, W, 1, 0.5)
    assert r.achieved_sparsity == 0.5 and r.total_damage == 1.0
    assert list(r.bias) == [-2.0, -2.0]
    r = _calib(S, W, 1, 0.1)
    assert r.total_damage == 0.0 and r.achieved_sparsity == 0.375
    assert list(r.bias) == [-1.0, -2.0]
    r = _calib(S, W, 1, 1.0)
    assert r.achieved_sparsity == 1.0 and r.total_damage == 17.0 and r.bias[0] == -4.0
    for bad in (0.0, 1.5):
        with pytest.raises(DataError):
            _calib(S, W, 1, bad)
    r = _calib([[1, 2], [1, 2]], [[1, 1], [1, 1]], 1, 0.25)  # ties -> lowest neuron index
    assert r.bias[0] == -1.0 and r.bias[1] == np.inf
    r = _calib([[1, 2, 3, 4]], [[1, 1, 1, 1]], 8, 0.25)  # step clamps at T
    assert r.achieved_sparsity == 1.0 and r.total_damage == 4.0
    r = _calib([[1, 2, 3], [1, 2, 3]], [[0, 0, 0], [1, 1, 1]], 1, 0.5)
    assert r.total_damage == 0.0 and r.bias[0] == -3.0
    r = _calib([[1, 1, 1, 1]], [[0, 1, 2, 3]], 1, 0.5)  # score ties drop together
    assert r.achieved_sparsity == 1.0 and r.total_damage == 0.0 and r.bias[0] == -1.0
    r = _calib([[1, 2, 3, 4], [1, 2, 3, 4]], [[1, 1, 1, 1], [5, 5, 5, 5]], 1, 0.25)
    assert r.bias[1] == np.inf and r.total_damage == 2.0
    with pytest.raises(DataError):
        _calib([[1]], [[-1]], 1, 0.5)  # negative weights


def test_layer_create_rejects_bad_descriptors_without_gpu():
    """Argument validation runs before any device work (types.hpp:31-51, :82-105)."""
    from paper_2603_14110_b200 import DeviceLayer, FfnWeights
    with pytest.raises(UsageError):
        DeviceLayer()
    with pytest.raises(DataError):
        DeviceLayer(FfnWeights(np.zeros((4, 2)), np.zeros((4, 2)), np.zeros((3, 4))))
