"""Tensor file format and the `run` document — the data formats on either
side of the executor.

``TensorValue`` mirrors the reference's tensor file unit (interp.py:34-70):
``{"dtype": "f64"|"i64"|"i32"|"bool", "shape": [...], "data": [row-major
items]}``.  ``run_document`` mirrors the non-distributed branch of the
reference's ``run`` command (cli.py:155-188): load a serialized graph (schema
v1) and one tensor file per non-transient container, execute, and return
``{"outputs": {name: tensor}, "report": {"per_rank": {0: counters}}}`` — here
executed by the B200 backend.  Errors follow the reference's exit codes: 1
for a missing input tensor, 2 for runtime errors.
"""

from __future__ import annotations

import json
import pathlib
from dataclasses import dataclass

import numpy as np

from . import sdfg

_NP = {"f64": np.float64, "i64": np.int64, "i32": np.int32, "bool": np.bool_}


@dataclass
class TensorValue:
    """Shape + row-major payload (interp.py:34-70)."""

    dtype: str
    array: np.ndarray

    @staticmethod
    def of(array, dtype: str | None = None) -> "TensorValue":
        arr = np.asarray(array)
        if dtype is None:
            kind = arr.dtype.kind
            dtype = "f64" if kind == "f" else ("i64" if kind in "iu" else "bool")
        if dtype not in _NP:
            raise ValueError(f"unknown dtype '{dtype}'")
        return TensorValue(dtype, np.ascontiguousarray(arr.astype(_NP[dtype])))

    def to_json(self) -> dict:
        return {"dtype": self.dtype, "shape": list(self.array.shape),
                "data": [x.item() for x in self.array.reshape(-1)]}

    @staticmethod
    def from_json(doc: dict) -> "TensorValue":
        dt = doc["dtype"]
        if dt not in _NP:
            raise ValueError(f"unknown dtype '{dt}'")
        return TensorValue(dt, np.array(doc["data"], dtype=_NP[dt]).reshape(doc["shape"]))

    @staticmethod
    def load(path) -> "TensorValue":
        with open(path) as f:
            return TensorValue.from_json(json.load(f))

    def save(self, path) -> None:
        with open(path, "w") as f:
            json.dump(self.to_json(), f, indent=1)
            f.write("\n")


class RunError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def run_document(graph, bindings: dict, inputs_dir, options=None) -> dict:
    """Execute a serialized graph on the GPU with inputs from tensor files
    (cli.py:155-188, non-distributed branch).  Raises RunError(1) for a
    missing input tensor and RunError(2) for executor errors."""
    from .machine import ExecContext, InterpreterError, interpret

    g = sdfg.as_graph(graph) if not isinstance(graph, (str, pathlib.Path)) else sdfg.load(graph)
    ctx = ExecContext(bindings=dict(bindings))
    d = pathlib.Path(inputs_dir) if inputs_dir is not None else None
    for name, desc in g.containers.items():
        if desc.transient:
            continue
        if d is not None and (d / f"{name}.json").exists():
            ctx.store[name] = TensorValue.load(d / f"{name}.json").array
        else:
            raise RunError(1, f"missing input tensor for '{name}'")
    try:
        outputs = interpret(g, ctx, options)
    except InterpreterError as ex:
        raise RunError(2, f"runtime error: {ex}") from ex
    return {"outputs": {k: TensorValue.of(v).to_json() for k, v in outputs.items()},
            "report": {"per_rank": {0: ctx.counters.as_dict()}}}
