"""The reference's tensor container (proj/include/sparsegate/tensor_io.hpp), so a
reference user's saved weights, predictors and activation batches load here.

A container is a directory with ``manifest.json`` (``{"entries": [{name, dtype,
shape, file, layout: "row-major", endianness: "little"}]}``) and one raw
little-endian row-major file per tensor. Reading and writing follow
tensor_io.hpp:73-331 (same checks, same IoError cases, files named
``<entry>.bin``, manifest written last).

Extension, rejected by the reference's reader by design:
dtype ``"bf16"`` (uint16 bit patterns) and the device-layer container
(``save_device_layer`` / ``load_device_layer``) holding exactly what
sg_layer_create uploads — bf16 gate, up, neuron-major ``down_t``, A, B and an
f32 bias — so a prepared layer reloads without the f64 -> bf16 pass.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .ffn_exec import (Activation, DataError, FfnWeights, IoError, Predictor, validate_predictor,
                       validate_weights)

_DT = {"f32": np.dtype("<f4"), "f64": np.dtype("<f8"), "bf16": np.dtype("<u2")}


@dataclass
class TensorEntry:  # tensor_io.hpp:34-47
    name: str
    dtype: str
    shape: List[int]
    file: str

    def elements(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n


@dataclass
class TensorManifest:  # tensor_io.hpp:49-70
    dir: str
    entries: List[TensorEntry] = field(default_factory=list)

    def find(self, name: str) -> Optional[TensorEntry]:
        for e in self.entries:
            if e.name == name:
                return e
        return None

    def at(self, name: str) -> TensorEntry:
        e = self.find(name)
        if e is None:
            raise IoError(f'container {self.dir}: missing entry "{name}"')
        return e


def load_manifest(directory: str, allow_ext: bool = True) -> TensorManifest:
    """tensor_io.hpp:73-138: parse manifest.json, check sizes against the files."""
    path = os.path.join(directory, "manifest.json")
    try:
        with open(path, "rb") as f:
            doc = json.loads(f.read().decode("utf-8"))
    except FileNotFoundError:
        raise IoError(f"cannot open {path}") from None
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise IoError(f"malformed manifest {path}: {e}") from None
    m = TensorManifest(directory)
    try:
        for je in doc["entries"]:
            name = je["name"]
            dtype = je["dtype"]
            if dtype not in _DT or (dtype == "bf16" and not allow_ext):
                raise IoError(f'manifest: unknown dtype "{dtype}"')
            shape = []
            for s in je["shape"]:
                if not isinstance(s, int) or isinstance(s, bool):
                    raise IoError(f'malformed manifest {path}: shape of "{name}"')
                if s < 0:
                    raise IoError(f'manifest: negative extent in shape of "{name}"')
                shape.append(s)
            file = je["file"]
            if je["layout"] != "row-major":
                raise IoError(f'manifest: entry "{name}" has unsupported layout')
            if je["endianness"] != "little":
                raise IoError(f'manifest: entry "{name}" has unsupported endianness')
            m.entries.append(TensorEntry(name, dtype, shape, file))
    except (KeyError, TypeError) as e:
        raise IoError(f"malformed manifest {path}: {e}") from None
    names = [e.name for e in m.entries]
    for i, n in enumerate(names):
        if n in names[i + 1:]:
            raise IoError(f'manifest: duplicate entry name "{n}"')
    for e in m.entries:
        f = os.path.join(directory, e.file)
        try:
            actual = os.path.getsize(f)
        except OSError:
            raise IoError(f"container: cannot stat {f}") from None
        expected = e.elements() * _DT[e.dtype].itemsize
        if actual != expected:
            raise IoError(f'container: entry "{e.name}" declares {expected} bytes but {f} has {actual}')
    return m


def read_payload(m: TensorManifest, e: TensorEntry, raw: bool = False) -> np.ndarray:
    """tensor_io.hpp:142-163 (f32 widened to f64; bf16 returned as uint16 when raw)."""
    f = os.path.join(m.dir, e.file)
    try:
        data = np.fromfile(f, dtype=_DT[e.dtype], count=e.elements())
    except OSError:
        raise IoError(f"cannot open {f}") from None
    if data.size != e.elements():
        raise IoError(f"short read on {f}")
    if e.dtype == "bf16":
        if raw:
            return data.reshape(e.shape)
        from .ffn_exec import bf16_to_f64
        return bf16_to_f64(data).reshape(e.shape)
    return data.astype(np.float64).reshape(e.shape)


def load_matrix(m: TensorManifest, name: str) -> np.ndarray:  # tensor_io.hpp:187-197
    e = m.at(name)
    if len(e.shape) != 2:
        raise IoError(f'entry "{name}": expected rank-2 tensor, got rank {len(e.shape)}')
    return read_payload(m, e)


def load_vector(m: TensorManifest, name: str) -> np.ndarray:  # tensor_io.hpp:199-209
    e = m.at(name)
    if len(e.shape) != 1:
        raise IoError(f'entry "{name}": expected rank-1 tensor, got rank {len(e.shape)}')
    return read_payload(m, e)


class ContainerWriter:
    """tensor_io.hpp:214-265: `<entry>.bin` payloads, manifest written last."""

    def __init__(self, directory: str):
        self.dir = directory
        os.makedirs(directory, exist_ok=True)
        self.entries: List[TensorEntry] = []

    def add(self, name: str, data, dtype: str = "f64") -> None:
        if dtype not in _DT:
            raise IoError(f'unknown dtype "{dtype}"')
        a = np.asarray(data)
        arr = np.ascontiguousarray(a, dtype=_DT[dtype]) if dtype != "bf16" else \
            np.ascontiguousarray(a, dtype=np.uint16)
        e = TensorEntry(name, dtype, list(a.shape), name + ".bin")
        try:
            arr.astype(_DT[dtype], copy=False).tofile(os.path.join(self.dir, e.file))
        except OSError:
            raise IoError(f"cannot create {os.path.join(self.dir, e.file)}") from None
        self.entries.append(e)

    def finish(self) -> None:
        doc = {"entries": [{"name": e.name, "dtype": e.dtype, "shape": e.shape, "file": e.file,
                            "layout": "row-major", "endianness": "little"} for e in self.entries]}
        with open(os.path.join(self.dir, "manifest.json"), "w") as f:
            f.write(json.dumps(doc, indent=2) + "\n")


# ---- typed containers (tensor_io.hpp:267-331) ----
def load_ffn_weights(m: TensorManifest, activation: Activation = Activation.ReGLU) -> FfnWeights:
    w = FfnWeights(load_matrix(m, "gate"), load_matrix(m, "up"), load_matrix(m, "down"), activation)
    validate_weights(w)
    return w


def save_ffn_weights(w: FfnWeights, directory: str, dtype: str = "f64") -> None:
    validate_weights(w)
    wr = ContainerWriter(directory)
    wr.add("gate", w.gate, dtype)
    wr.add("up", w.up, dtype)
    wr.add("down", w.down, dtype)
    wr.finish()


def load_activation_batch(m: TensorManifest, name: str = "x") -> np.ndarray:
    x = load_matrix(m, name)  # d x N, tokens as columns; N = 0 is representable
    if not np.all(np.isfinite(x)):
        raise IoError(f'activation batch "{name}": non-finite entries')
    return x


def save_activation_batch(x_cols, directory: str, dtype: str = "f64", name: str = "x") -> None:
    wr = ContainerWriter(directory)
    wr.add(name, np.asarray(x_cols, dtype=np.float64), dtype)
    wr.finish()


def save_predictor(p: Predictor, directory: str) -> None:  # always f64: byte-exact round trip
    validate_predictor(p)
    wr = ContainerWriter(directory)
    wr.add("A", p.A, "f64")
    wr.add("B", p.B, "f64")
    wr.add("bias", p.bias, "f64")
    wr.finish()


def load_predictor(directory: str) -> Predictor:
    m = load_manifest(directory)
    A, B, bias = load_matrix(m, "A"), load_matrix(m, "B"), load_vector(m, "bias")
    p = Predictor(A, B, bias, A.shape[1])
    validate_predictor(p)
    return p


# ---- extension: the device-layer container ----
def save_device_layer(directory: str, hidden: int, inter: int, activation: int, gate, up, down_t,
                      A=None, B=None, bias=None, order=None) -> None:
    """bf16 (uint16) gate / up / down_t (inter x hidden, neuron-major), A, B; f32 bias;
    optional int64-as-f64 layout order. Loads with load_device_layer."""
    wr = ContainerWriter(directory)
    for name, arr in (("gate", gate), ("up", up), ("down_t", down_t)):
        a = np.asarray(arr)
        if a.dtype != np.uint16 or a.shape != (inter, hidden):
            raise DataError(f"device layer: {name} must be uint16 (bf16) {inter} x {hidden}")
        wr.add(name, a, "bf16")
    if A is not None:
        wr.add("A", np.asarray(A, dtype=np.uint16), "bf16")
        wr.add("B", np.asarray(B, dtype=np.uint16), "bf16")
        wr.add("bias", np.asarray(bias, dtype=np.float32), "f32")
    if order is not None:
        wr.add("order", np.asarray(order, dtype=np.float64), "f64")
    wr.add("meta", np.array([hidden, inter, activation], dtype=np.float64), "f64")
    wr.finish()


def load_device_layer(directory: str, device: int = 0, shard_index: int = 0, shard_count: int = 1):
    """-> DeviceLayer uploaded straight from the bf16 container."""
    from .ffn_exec import DeviceLayer
    m = load_manifest(directory)
    hidden, inter, act = (int(v) for v in load_vector(m, "meta"))
    raw = dict(hidden=hidden, inter=inter, activation=act,
               gate=read_payload(m, m.at("gate"), raw=True),
               up=read_payload(m, m.at("up"), raw=True),
               down_t=read_payload(m, m.at("down_t"), raw=True))
    if m.find("A") is not None:
        A = read_payload(m, m.at("A"), raw=True)
        raw.update(rank=int(A.shape[1]), A=A, B=read_payload(m, m.at("B"), raw=True),
                   bias=read_payload(m, m.at("bias")).astype(np.float32))
    if m.find("order") is not None:
        raw["order"] = load_vector(m, "order").astype(np.int64)
    return DeviceLayer(raw=raw, device=device, shard_index=shard_index, shard_count=shard_count)
