#!/usr/bin/env python
"""Generate the golden vectors in tests/golden/ from the REAL reference executor.

The reference headers (/root/reference/proj/include/sparsegate/*.hpp) are
compiled unmodified into oracle/_ref/libsgref.so (oracle/Makefile); this script
drives them through the reference's own RNG streams (std::mt19937_64 +
std::normal_distribution, exactly as proj/tests/ffn_exec_tests.cpp and
proj/tests/test_support.hpp draw them) and stores inputs and outputs.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The .npz files are committed; tests/test_oracle.py checks the f64 restatement
(oracle/sg_oracle.cpp) against them on any machine.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def random_ffn(rng, d, D):
    """ffn_exec_tests.cpp:16-24 (random_matrix order: gate, up, down)."""
    gate = rng.random_matrix(D, d)
    up = rng.random_matrix(D, d)
    down = rng.random_matrix(d, D)
    return gate, up, down


def run_all(gate, up, down, A, B, bias, x, act, rank_field=None):
    out = {}
    y, st = O.ref_dense_ffn(gate, up, down, x, act)
    out["dense_y"] = y
    out["dense_mult"] = st.multiplies
    for name, pipe in (("par", 1), ("seq", 2)):
        y, st = O.ref_sparse_ffn(gate, up, down, A, B, bias, x, act, pipe, rank_field)
        out[f"{name}_y"] = y
        out[f"{name}_mult"] = st.multiplies
        out[f"{name}_ps"] = st.predicted_sparsity
        out[f"{name}_rs"] = st.realized_sparsity
    mask, cnt = O.ref_predict_mask(A, B, bias, x, rank_field)
    out["mask"] = mask
    out["count"] = cnt
    return out


def save(name, **arrs):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrs)


def stack_trials(trials):
    keys = trials[0].keys()
    return {k: np.array([t[k] for t in trials]) for k in keys}


def main():
    if not O.ref_available():
        O.build()
    # ffn_exec_tests.cpp:51-82 — 2x2 known answers
    gate = np.array([[1.0, 0.0], [-1.0, 0.0]])
    eye = np.eye(2)
    y, st = O.ref_dense_ffn(gate, eye, eye, np.array([1.0, 1.0]))
    y0, _ = O.ref_dense_ffn(gate, eye, eye, np.zeros(2))
    up2 = np.array([[-1.0, 0.0], [0.0, 1.0]])
    yr, _ = O.ref_dense_ffn(gate, up2, eye, np.array([1.0, 1.0]), 0)
    yd, _ = O.ref_dense_ffn(gate, up2, eye, np.array([1.0, 1.0]), 1)
    save("dense_2x2", gate=gate, y=y, mult=st.multiplies, y_zero=y0, up2=up2, y_reglu=yr,
         y_drelu=yd)

    # ffn_exec_tests.cpp:84-99 — exact predictor mask (seed 13)
    rng = O.RefRng(13)
    g, u, dn = random_ffn(rng, 8, 24)
    xs = np.stack([rng.random_vector(8) for _ in range(10)])
    masks, counts = [], []
    for x in xs:
        m, cn = O.ref_predict_mask(g, np.eye(8), np.zeros(24), x)
        masks.append(m)
        counts.append(cn)
    save("mask_exact_seed13", gate=g, up=u, down=dn, xs=xs, masks=np.array(masks),
         counts=np.array(counts))

    # ffn_exec_tests.cpp:124-138 — all-active (seed 29), both activations
    rng = O.RefRng(29)
    cases = {}
    for act in (0, 1):
        g, u, dn = random_ffn(rng, 16, 48)
        xs = np.stack([rng.random_vector(16) for _ in range(5)])
        trials = [run_all(g, u, dn, g, np.eye(16), np.full(48, 1e12), x, act) for x in xs]
        cases.update({f"a{act}_gate": g, f"a{act}_up": u, f"a{act}_down": dn, f"a{act}_xs": xs})
        cases.update({f"a{act}_{k}": v for k, v in stack_trials(trials).items()})
    save("all_active_seed29", **cases)

    # ffn_exec_tests.cpp:140-153 — all-off (seed 31)
    rng = O.RefRng(31)
    g, u, dn = random_ffn(rng, 8, 24)
    x = rng.random_vector(8)
    r = run_all(g, u, dn, g, np.eye(8), np.full(24, -1e12), x, 0)
    save("all_off_seed31", gate=g, up=u, down=dn, x=x, **r)

    # ffn_exec_tests.cpp:155-169 — perfect recall (seed 37)
    rng = O.RefRng(37)
    cases = {}
    for trial in range(20):
        act = trial % 2
        g, u, dn = random_ffn(rng, 12, 40)
        x = rng.random_vector(12)
        r = run_all(g, u, dn, g, np.eye(12), np.zeros(40), x, act)
        cases.update({f"t{trial}_gate": g, f"t{trial}_up": u, f"t{trial}_down": dn,
                      f"t{trial}_x": x})
        cases.update({f"t{trial}_{k}": v for k, v in r.items()})
    save("perfect_recall_seed37", **cases)

    # ffn_exec_tests.cpp:171-192 — revalidation (seed 41)
    rng = O.RefRng(41)
    g, u, dn = random_ffn(rng, 8, 32)
    x = rng.random_vector(8)
    r = run_all(g, u, dn, g, np.eye(8), np.full(32, 1e12), x, 0)
    save("revalidation_seed41", gate=g, up=u, down=dn, x=x, **r)

    # ffn_exec_tests.cpp:194-230 — random-bias predictors (seeds 43, 47)
    rng = O.RefRng(43)
    cases = {}
    for trial in range(20):
        g, u, dn = random_ffn(rng, 8, 24)
        bias = rng.random_vector(24)
        x = rng.random_vector(8)
        r = run_all(g, u, dn, g, np.eye(8), bias, x, 0)
        cases.update({f"t{trial}_gate": g, f"t{trial}_up": u, f"t{trial}_down": dn,
                      f"t{trial}_bias": bias, f"t{trial}_x": x})
        cases.update({f"t{trial}_{k}": v for k, v in r.items()})
    save("random_bias_seed43", **cases)
    rng = O.RefRng(47)
    g, u, dn = random_ffn(rng, 8, 24)
    bias = rng.random_vector(24)
    x = rng.random_vector(8)
    save("multiply_model_seed47", gate=g, up=u, down=dn, bias=bias, x=x,
         **run_all(g, u, dn, g, np.eye(8), bias, x, 0))

    # ffn_exec_tests.cpp:232-254 — determinism (seed 53)
    rng = O.RefRng(53)
    g, u, dn = random_ffn(rng, 16, 64)
    bias = rng.random_vector(64)
    x = rng.random_vector(16)
    save("determinism_seed53", gate=g, up=u, down=dn, bias=bias, x=x,
         **run_all(g, u, dn, g, np.eye(16), bias, x, 0))

    # ffn_exec_tests.cpp:256-279 — op-count model
    ops = []
    for args in ((4096, 11008, 256, 0.5, 0.9), (64, 256, 0, 0.0, 0.0), (64, 256, 8, 1.0, 1.0)):
        ops.append(list(args) + list(O.ref_op_count_model(*args)))
    save("op_count", rows=np.array(ops, dtype=np.float64))

    # synthetic.hpp:80-108 — fixture stream (acceptance_main.cpp:249-258 shape, seed 9)
    f = O.ref_synthetic(32, 128, 128, 32, 0.9, 9)
    save("synthetic_h32_i128_s9", **f)
    # a mid-size executor case on synthetic weights with a low-rank random predictor
    f = O.ref_synthetic(64, 256, 8, 6, 0.9, 21)
    rng = O.RefRng(2101)
    A = rng.random_matrix(256, 16, 0.3)
    B = rng.random_matrix(16, 64, 0.3)
    bias = rng.random_vector(256, 0.5)
    cases = {"gate": f["gate"], "up": f["up"], "down": f["down"], "A": A, "B": B, "bias": bias,
             "xs": f["eval"].T.copy()}
    for act in (0, 1):
        trials = [run_all(f["gate"], f["up"], f["down"], A, B, bias, x, act) for x in f["eval"].T]
        cases.update({f"a{act}_{k}": v for k, v in stack_trials(trials).items()})
    save("synthetic_exec_h64_i256_r16", **cases)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
