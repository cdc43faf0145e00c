"""CPU: the f64 oracle (oracle/sg_oracle.cpp) pinned against the reference.

1. Golden vectors produced by the real reference headers (tests/golden/, made
   by tests/golden/make_golden.py from oracle/_ref/libsgref.so) must be
   reproduced bit-for-bit by the restatement.
2. The reference's own known answers and properties
   (/root/reference/proj/tests/ffn_exec_tests.cpp) hold in the goldens.
3. Where oracle/_ref exists (built from /root/reference in this container),
   restatement == reference bit-for-bit on fresh random instances too.
"""
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def check_all(gate, up, down, A, B, bias, x, act, exp, prefix=""):
    y, st = O.dense_ffn(gate, up, down, x, act)
    assert np.array_equal(y, exp[prefix + "dense_y"])
    assert st.multiplies == exp[prefix + "dense_mult"]
    for name, pipe in (("par", 1), ("seq", 2)):
        o = O.sparse_ffn(gate, up, down, A, B, bias, x, act, pipe)
        assert np.array_equal(o.y, exp[prefix + f"{name}_y"]), name
        assert o.stats.multiplies == exp[prefix + f"{name}_mult"]
        assert o.stats.predicted_sparsity == exp[prefix + f"{name}_ps"]
        assert o.stats.realized_sparsity == exp[prefix + f"{name}_rs"]
    mask, cnt, _ = O.predict_mask(A, B, bias, x)
    assert np.array_equal(mask, exp[prefix + "mask"]) and cnt == exp[prefix + "count"]


def test_dense_2x2_known_answer():  # ffn_exec_tests.cpp:51-82
    g = load("dense_2x2")
    eye = np.eye(2)
    y, st = O.dense_ffn(g["gate"], eye, eye, [1.0, 1.0])
    assert np.array_equal(y, g["y"]) and list(y) == [1.0, 0.0] and st.multiplies == 12
    assert np.array_equal(O.dense_ffn(g["gate"], eye, eye, np.zeros(2))[0], g["y_zero"])
    assert O.dense_ffn(g["gate"], g["up2"], eye, [1.0, 1.0], 0)[0][0] == g["y_reglu"][0] == -1.0
    assert O.dense_ffn(g["gate"], g["up2"], eye, [1.0, 1.0], 1)[0][0] == g["y_drelu"][0] == 0.0
    with pytest.raises(O.OracleError) as e:
        O.dense_ffn(g["gate"], eye, eye, [1.0, np.nan])
    assert e.value.code == 2  # DataError


def test_exact_predictor_mask_seed13():  # ffn_exec_tests.cpp:84-99
    g = load("mask_exact_seed13")
    for x, m, c in zip(g["xs"], g["masks"], g["counts"]):
        mask, cnt, _ = O.predict_mask(g["gate"], np.eye(8), np.zeros(24), x)
        assert np.array_equal(mask, m) and cnt == c
        gp = np.array([O.det_dot(g["gate"][i], x) for i in range(24)])
        assert np.array_equal(mask.astype(bool), gp > 0)


def test_zero_preactivation_inactive_and_constant_bias():  # ffn_exec_tests.cpp:101-121
    m, c, _ = O.predict_mask(np.array([[1.0, -1.0], [1.0, 0.0]]), np.eye(2), np.zeros(2), [1, 1])
    assert list(m) == [0, 1] and c == 1
    g = load("mask_exact_seed13")
    x = g["xs"][0]
    assert O.predict_mask(g["gate"], np.eye(8), np.full(24, 1e12), x)[1] == 24
    assert O.predict_mask(g["gate"], np.eye(8), np.full(24, -1e12), x)[1] == 0


@pytest.mark.parametrize("act", [0, 1])
def test_all_active_seed29(act):  # ffn_exec_tests.cpp:124-138
    g = load("all_active_seed29")
    p = f"a{act}_"
    for t, x in enumerate(g[p + "xs"]):
        exp = {k[len(p):]: v[t] for k, v in g.items() if k.startswith(p) and k != p + "xs"
               and k not in (p + "gate", p + "up", p + "down")}
        check_all(g[p + "gate"], g[p + "up"], g[p + "down"], g[p + "gate"], np.eye(16),
                  np.full(48, 1e12), x, act, exp)
        assert np.array_equal(exp["par_y"], exp["dense_y"])  # reference property
        assert np.array_equal(exp["seq_y"], exp["dense_y"])


def test_all_off_seed31():  # ffn_exec_tests.cpp:140-153
    g = load("all_off_seed31")
    check_all(g["gate"], g["up"], g["down"], g["gate"], np.eye(8), np.full(24, -1e12), g["x"], 0, g)
    assert np.all(g["seq_y"] == 0) and g["seq_mult"] == 8 * (8 + 24)
    assert g["seq_ps"] == 1.0 and g["seq_rs"] == 1.0


def test_perfect_recall_seed37():  # ffn_exec_tests.cpp:155-169
    g = load("perfect_recall_seed37")
    for t in range(20):
        p = f"t{t}_"
        exp = {k[len(p):]: v for k, v in g.items() if k.startswith(p)}
        check_all(exp["gate"], exp["up"], exp["down"], exp["gate"], np.eye(12), np.zeros(40),
                  exp["x"], t % 2, exp)
        scale = max(1e-300, np.linalg.norm(exp["dense_y"]))
        assert np.linalg.norm(exp["seq_y"] - exp["dense_y"]) <= 1e-12 * scale


def test_revalidation_seed41():  # ffn_exec_tests.cpp:171-192
    g = load("revalidation_seed41")
    check_all(g["gate"], g["up"], g["down"], g["gate"], np.eye(8), np.full(32, 1e12), g["x"], 0, g)
    support = sum(O.det_dot(g["gate"][i], g["x"]) > 0 for i in range(32))
    assert support < 32
    assert np.array_equal(g["seq_y"], g["par_y"])
    assert g["seq_mult"] == 8 * (8 + 32) + 8 * 32 + 2 * 8 * support
    assert g["seq_rs"] > g["seq_ps"]


def test_random_bias_seed43_and_model_seed47():  # ffn_exec_tests.cpp:194-230
    g = load("random_bias_seed43")
    for t in range(20):
        p = f"t{t}_"
        exp = {k[len(p):]: v for k, v in g.items() if k.startswith(p)}
        check_all(exp["gate"], exp["up"], exp["down"], exp["gate"], np.eye(8), exp["bias"],
                  exp["x"], 0, exp)
        assert exp["seq_rs"] >= exp["seq_ps"]
    g = load("multiply_model_seed47")
    check_all(g["gate"], g["up"], g["down"], g["gate"], np.eye(8), g["bias"], g["x"], 0, g)
    p = int(g["count"])
    v = sum(1 for i in range(24) if g["mask"][i] and O.det_dot(g["gate"][i], g["x"]) > 0)
    assert g["dense_mult"] == 3 * 8 * 24
    assert g["par_mult"] == 8 * (8 + 24) + 3 * 8 * p
    assert g["seq_mult"] == 8 * (8 + 24) + 8 * p + 2 * 8 * v


def test_determinism_seed53():  # ffn_exec_tests.cpp:232-254
    g = load("determinism_seed53")
    check_all(g["gate"], g["up"], g["down"], g["gate"], np.eye(16), g["bias"], g["x"], 0, g)
    assert np.array_equal(g["par_y"], g["seq_y"])


def test_op_count_model():  # ffn_exec_tests.cpp:256-279
    rows = load("op_count")["rows"]
    for r in rows:
        d, D, r_, s, sp, dense, sparse, ratio = r
        got = O.op_count_model(int(d), int(D), int(r_), s, sp)
        assert got == (int(dense), sparse, ratio)
    dense, sparse, ratio = O.op_count_model(4096, 11008, 256, 0.5, 0.9)
    assert dense == 135266304 and abs(sparse - 35428761.6) < 1e-6 and f"{ratio:.2f}" == "3.82"
    with pytest.raises(O.OracleError):
        O.op_count_model(64, 256, 8, 0.9, 0.5)


def test_synthetic_stream_seed9():  # synthetic.hpp:80-108
    g = load("synthetic_h32_i128_s9")
    f = O.synthetic(32, 128, 128, 32, 0.9, 9)
    for k in ("gate", "up", "down", "calib", "eval"):
        assert np.array_equal(f[k], g[k]), k


@pytest.mark.parametrize("act", [0, 1])
def test_synthetic_executor_h64(act):
    g = load("synthetic_exec_h64_i256_r16")
    p = f"a{act}_"
    for t, x in enumerate(g["xs"]):
        exp = {k[len(p):]: v[t] for k, v in g.items() if k.startswith(p)}
        check_all(g["gate"], g["up"], g["down"], g["A"], g["B"], g["bias"], x, act, exp)


def test_index_sets_are_consistent():
    """The restatement's extra outputs: P == mask support, V == {i in P: g_i > 0}."""
    g = load("synthetic_exec_h64_i256_r16")
    for x in g["xs"]:
        o = O.sparse_ffn(g["gate"], g["up"], g["down"], g["A"], g["B"], g["bias"], x)
        mask, _, _ = O.predict_mask(g["A"], g["B"], g["bias"], x)
        assert np.array_equal(o.P, np.nonzero(mask)[0])
        gv = np.array([O.det_dot(g["gate"][i], x) for i in o.P])
        assert np.array_equal(o.V, o.P[gv > 0])
        assert np.array_equal(o.g, gv)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_restatement_matches_live_reference(seed):
    rng = np.random.default_rng(seed)
    d, D, r = 24, 72, 6
    gate, up, down = rng.standard_normal((D, d)), rng.standard_normal((D, d)), rng.standard_normal((d, D))
    A, B, bias = rng.standard_normal((D, r)), rng.standard_normal((r, d)), rng.standard_normal(D)
    bias[::7] = np.inf
    for act in (0, 1):
        for _ in range(3):
            x = rng.standard_normal(d)
            for pipe in (1, 2):
                y_ref, st_ref = O.ref_sparse_ffn(gate, up, down, A, B, bias, x, act, pipe)
                o = O.sparse_ffn(gate, up, down, A, B, bias, x, act, pipe)
                assert np.array_equal(o.y, y_ref)
                assert (o.stats.multiplies, o.stats.predicted_sparsity, o.stats.realized_sparsity) == \
                    (st_ref.multiplies, st_ref.predicted_sparsity, st_ref.realized_sparsity)
            assert np.array_equal(O.dense_ffn(gate, up, down, x, act)[0],
                                  O.ref_dense_ffn(gate, up, down, x, act)[0])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_reference_error_taxonomy():
    """types.hpp validation errors surface as DataError (code 2) in both."""
    rng = np.random.default_rng(0)
    gate = rng.standard_normal((8, 4))
    with pytest.raises(O.OracleError) as e1:
        O.ref_sparse_ffn(gate, gate, gate.T, gate[:, :2], rng.standard_normal((2, 4)), np.zeros(8),
                         np.ones(4), rank_field=3)
    with pytest.raises(O.OracleError) as e2:
        O.sparse_ffn(gate, gate, gate.T, gate[:, :2], rng.standard_normal((2, 4)), np.zeros(8),
                     np.ones(4), rank_field=3)
    assert e1.value.code == e2.value.code == 2
