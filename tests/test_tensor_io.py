"""CPU: the tensor container (paper_2603_14110_b200/tensor_io.py) behaves like
the reference's tensor_io.hpp — the cases of proj/tests/tensor_io_tests.cpp."""
import json
import os

import numpy as np
import pytest

from paper_2603_14110_b200 import Activation, DataError, FfnWeights, IoError, Predictor
from paper_2603_14110_b200 import tensor_io as T


def write_manifest(d, entries):
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "manifest.json"), "w") as f:
        json.dump({"entries": entries}, f)


def entry(name, dtype="f64", shape=(3, 4), file=None, layout="row-major", endianness="little"):
    return dict(name=name, dtype=dtype, shape=list(shape), file=file or name + ".bin",
                layout=layout, endianness=endianness)


def test_manifest_parses_and_checks_sizes(tmp_path):  # tensor_io_tests.cpp:13-34
    d = str(tmp_path)
    np.zeros(12).tofile(os.path.join(d, "gate.bin"))
    write_manifest(d, [entry("gate")])
    m = T.load_manifest(d)
    assert m.entries[0].name == "gate" and m.entries[0].dtype == "f64" and m.entries[0].elements() == 12
    np.zeros(11).tofile(os.path.join(d, "gate.bin"))
    with pytest.raises(IoError):
        T.load_manifest(d)


def test_empty_manifest_is_valid(tmp_path):  # :36-40
    write_manifest(str(tmp_path), [])
    assert T.load_manifest(str(tmp_path)).entries == []


@pytest.mark.parametrize("case", ["missing", "malformed", "dtype", "dup", "nofile", "layout",
                                  "endian", "negative"])
def test_manifest_failure_modes(tmp_path, case):  # :42-73 (+ layout / endianness / extent)
    d = str(tmp_path)
    np.zeros(12).tofile(os.path.join(d, "g.bin"))
    if case == "missing":
        with pytest.raises(IoError):
            T.load_manifest(os.path.join(d, "nope"))
        return
    if case == "malformed":
        with open(os.path.join(d, "manifest.json"), "w") as f:
            f.write("{ not json")
    elif case == "dtype":
        write_manifest(d, [entry("g", dtype="f16")])
    elif case == "dup":
        write_manifest(d, [entry("g"), entry("g")])
    elif case == "nofile":
        write_manifest(d, [entry("h")])
    elif case == "layout":
        write_manifest(d, [entry("g", layout="col-major")])
    elif case == "endian":
        write_manifest(d, [entry("g", endianness="big")])
    elif case == "negative":
        write_manifest(d, [entry("g", shape=(-3, -4))])
    with pytest.raises(IoError):
        T.load_manifest(d)


def test_f32_payload_declared_f64_fails_by_size(tmp_path):  # :75-90
    d = str(tmp_path)
    np.zeros(12, dtype=np.float32).tofile(os.path.join(d, "g.bin"))
    write_manifest(d, [entry("g", dtype="f64")])
    with pytest.raises(IoError):
        T.load_manifest(d)


def test_ffn_weights_round_trip_and_shape_checks(tmp_path):  # :92-125
    rng = np.random.default_rng(0)
    w = FfnWeights(rng.standard_normal((2, 3)), rng.standard_normal((2, 3)), rng.standard_normal((3, 2)))
    d = str(tmp_path / "w")
    T.save_ffn_weights(w, d)
    got = T.load_ffn_weights(T.load_manifest(d), Activation.ReGLU)
    assert got.hidden_size() == 3 and got.inter_size() == 2
    assert np.array_equal(got.gate, w.gate) and np.array_equal(got.down, w.down)
    other = str(tmp_path / "o")
    wr = T.ContainerWriter(other)
    wr.add("gate", w.gate)
    wr.add("up", rng.standard_normal((3, 3)))
    wr.add("down", w.down)
    wr.finish()
    with pytest.raises(DataError):
        T.load_ffn_weights(T.load_manifest(other))
    with pytest.raises(DataError):
        T.save_ffn_weights(FfnWeights(w.gate, w.up, w.down.T.copy()), str(tmp_path / "bad"))
    os.remove(os.path.join(d, "up.bin"))
    with pytest.raises(IoError):
        T.load_manifest(d)


def test_predictor_round_trip_is_byte_exact(tmp_path):  # :127-142
    rng = np.random.default_rng(1)
    p = Predictor(rng.standard_normal((6, 3)), rng.standard_normal((3, 4)), rng.standard_normal(6), 3)
    p.bias[2] = np.inf
    d = str(tmp_path)
    T.save_predictor(p, d)
    q = T.load_predictor(d)
    assert q.A.tobytes() == p.A.tobytes() and q.B.tobytes() == p.B.tobytes()
    assert q.bias.tobytes() == p.bias.tobytes() and q.rank == 3


def test_predictor_container_errors(tmp_path):  # :144-163
    rng = np.random.default_rng(2)
    d = str(tmp_path / "a")
    wr = T.ContainerWriter(d)
    wr.add("A", rng.standard_normal((6, 3)))
    wr.add("B", rng.standard_normal((3, 4)))
    wr.finish()
    with pytest.raises(IoError):
        T.load_predictor(d)
    d2 = str(tmp_path / "b")
    wr = T.ContainerWriter(d2)
    wr.add("A", rng.standard_normal((6, 3)))
    wr.add("B", rng.standard_normal((2, 4)))
    wr.add("bias", rng.standard_normal(6))
    wr.finish()
    with pytest.raises(DataError, match="rank mismatch"):
        T.load_predictor(d2)


def test_container_round_trip_is_byte_identical(tmp_path):  # :165-190
    rng = np.random.default_rng(3)
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    wr = T.ContainerWriter(a)
    for i in range(4):
        wr.add(f"t{i}", rng.standard_normal((3, 5)), "f32" if i % 2 else "f64")
    wr.finish()
    m = T.load_manifest(a)
    wr = T.ContainerWriter(b)
    for e in m.entries:
        wr.add(e.name, T.read_payload(m, e), e.dtype)
    wr.finish()
    for e in m.entries:
        assert open(os.path.join(a, e.file), "rb").read() == open(os.path.join(b, e.file), "rb").read()
    assert open(os.path.join(a, "manifest.json")).read() == open(os.path.join(b, "manifest.json")).read()


def test_zero_token_batch_is_representable(tmp_path):  # :192-200
    T.save_activation_batch(np.zeros((4, 0)), str(tmp_path))
    x = T.load_activation_batch(T.load_manifest(str(tmp_path)))
    assert x.shape == (4, 0)


def test_bf16_extension_is_explicit(tmp_path):
    """bf16 entries are this repo's extension: accepted by default, rejected in strict mode."""
    d = str(tmp_path)
    wr = T.ContainerWriter(d)
    wr.add("g", np.arange(12, dtype=np.uint16).reshape(3, 4), "bf16")
    wr.finish()
    assert T.read_payload(T.load_manifest(d), T.load_manifest(d).at("g"), raw=True).dtype == np.uint16
    with pytest.raises(IoError):
        T.load_manifest(d, allow_ext=False)
