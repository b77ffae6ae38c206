"""Validation fixtures pinned to the REFERENCE's own validator.

Run here (the container with /root/reference), never on the GPU box:

    python tests/golden/make_validation_cases.py

Writes tests/golden/validation_cases.json: small schema-v1 graphs (hand
written here, in the style of pkg/tests/test_ir.py:15-110 — unordered
writes, parallel-map conflicts with and without WCR, disjoint / strided /
unprovable subsets, structural errors) together with the set of error codes
the reference's ``Sdfg.validate`` (pkg/src/sdfgkit/ir.py:595-745) reports for
each, after a round trip through its deserializer (serialize.py:238).
"""

from __future__ import annotations

import importlib
import json
import os
import pathlib
import sys

REF = pathlib.Path(os.environ.get("REF_PKG", "/root/reference/pkg"))
HERE = pathlib.Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF / "src"))
serialize = importlib.import_module("sdfgkit.serialize")


def arr(name, shape, transient=False, kind="array"):
    return {"name": name, "dtype": "f64", "shape": shape, "kind": kind, "transient": transient,
            "lifetime": "scope", "storage": "heap"}


def graph(name, containers, nodes, edges, symbols=("N",), transitions=(), states=None):
    st = states or [{"label": "s0", "nodes": nodes, "edges": edges}]
    return {"version": 1, "name": name, "symbols": [{"name": s, "min": 1} for s in symbols],
            "containers": containers, "states": st, "transitions": list(transitions),
            "start": st[0]["label"]}


def copy_writes(name, sub1, sub2, wcr1=None, wcr2=None, shape=("N",), symbols=("N",)):
    """Two tasklets writing x into A[sub1] and A[sub2] with no ordering path."""
    nodes, edges = [], []
    for k, (sub, w) in enumerate(((sub1, wcr1), (sub2, wcr2))):
        b = 3 * k
        nodes += [{"id": b, "type": "access", "container": "x"},
                  {"id": b + 1, "type": "tasklet", "name": f"w{k}", "ins": ["v"], "outs": ["out"],
                   "code": [["out", "v"]]},
                  {"id": b + 2, "type": "access", "container": "A"}]
        edges += [{"src": b, "dst": b + 1, "dst_conn": "v", "memlet": "x[]"}]
        e = {"src": b + 1, "dst": b + 2, "src_conn": "out", "memlet": f"A[{sub}]"}
        if w:
            e["wcr"] = w
        edges.append(e)
    return graph(name, [arr("A", list(shape)), arr("x", [], kind="scalar")], nodes, edges,
                 symbols=symbols)


def map_graph(name, rng, read, write, wcr=None, schedule="parallel", out_shape=None):
    """One map: tasklet reads A[read], writes B[write] (B scalar if shape [])."""
    out_shape = [] if out_shape is None else out_shape
    nodes = [{"id": 0, "type": "map_entry", "params": [["i", rng]], "schedule": schedule,
              "tiled": False},
             {"id": 1, "type": "map_exit", "entry": 0},
             {"id": 2, "type": "tasklet", "name": "t", "ins": ["v"], "outs": ["o"],
              "code": [["o", "v"]]},
             {"id": 3, "type": "access", "container": "A"},
             {"id": 4, "type": "access", "container": "B"}]
    w_outer = "B[]" if not out_shape else f"B[0:{out_shape[0]} - 1:1]"
    edges = [{"src": 3, "dst": 0, "dst_conn": "IN_v", "memlet": "A[0:N - 1:1]"},
             {"src": 0, "dst": 2, "src_conn": "OUT_v", "dst_conn": "v", "memlet": f"A[{read}]"},
             {"src": 2, "dst": 1, "src_conn": "o", "dst_conn": "IN_o", "memlet": f"B[{write}]"},
             {"src": 1, "dst": 4, "src_conn": "OUT_o", "memlet": w_outer}]
    if wcr:
        edges[2]["wcr"] = wcr
        edges[3]["wcr"] = wcr
    kind = "scalar" if not out_shape else "array"
    return graph(name, [arr("A", ["N"]), arr("B", out_shape, kind=kind)], nodes, edges)


def inplace_map(name, read, write):
    """A parallel map reading A[read] and writing A[write] (same container)."""
    nodes = [{"id": 0, "type": "map_entry", "params": [["i", "1:N - 2:1"]], "schedule": "parallel",
              "tiled": False},
             {"id": 1, "type": "map_exit", "entry": 0},
             {"id": 2, "type": "tasklet", "name": "t", "ins": ["v"], "outs": ["o"],
              "code": [["o", "v * 2.0"]]},
             {"id": 3, "type": "access", "container": "A"},
             {"id": 4, "type": "access", "container": "A"}]
    edges = [{"src": 3, "dst": 0, "dst_conn": "IN_v", "memlet": "A[0:N - 1:1]"},
             {"src": 0, "dst": 2, "src_conn": "OUT_v", "dst_conn": "v", "memlet": f"A[{read}]"},
             {"src": 2, "dst": 1, "src_conn": "o", "dst_conn": "IN_o", "memlet": f"A[{write}]"},
             {"src": 1, "dst": 4, "src_conn": "OUT_o", "memlet": "A[1:N - 2:1]"}]
    return graph(name, [arr("A", ["N"])], nodes, edges)


CASES = {
    "race_whole": copy_writes("race_whole", "0:N - 1:1", "0:N - 1:1"),
    "race_wcr_same": copy_writes("race_wcr_same", "0:N - 1:1", "0:N - 1:1", "add", "add"),
    "race_wcr_mixed": copy_writes("race_wcr_mixed", "0:N - 1:1", "0:N - 1:1", "add", "mul"),
    "disjoint_const": copy_writes("disjoint_const", "0:3:1", "4:7:1", shape=("8",)),
    "overlap_const": copy_writes("overlap_const", "0:4:1", "4:7:1", shape=("8",)),
    "disjoint_sym": copy_writes("disjoint_sym", "0:0:1", "1:N - 1:1"),
    "disjoint_stride": copy_writes("disjoint_stride", "0:N - 1:2", "1:N - 1:2"),
    "unprovable_sym": copy_writes("unprovable_sym", "0:N - 2:1", "N - 1:N - 1:1"),
    "unprovable_two_syms": copy_writes("unprovable_two_syms", "0:M - 1:1", "N - 1:N - 1:1",
                                       symbols=("N", "M")),
    "overlap_point": copy_writes("overlap_point", "N - 1:N - 1:1", "0:N - 1:1"),
    "map_conflict": map_graph("map_conflict", "0:N - 1:1", "i:i:1", ""),
    "map_conflict_wcr": map_graph("map_conflict_wcr", "0:N - 1:1", "i:i:1", "", wcr="add"),
    "map_conflict_seq": map_graph("map_conflict_seq", "0:N - 1:1", "i:i:1", "",
                                  schedule="sequential"),
    "map_pointwise": map_graph("map_pointwise", "0:N - 1:1", "i:i:1", "i:i:1", out_shape=["N"]),
    "map_shifted": map_graph("map_shifted", "0:N - 2:1", "i + 1:i + 1:1", "i:i:1",
                             out_shape=["N"]),
    "inplace_same_point": inplace_map("inplace_same_point", "i:i:1", "i:i:1"),
    "inplace_neighbour": inplace_map("inplace_neighbour", "i - 1:i - 1:1", "i:i:1"),
    "unknown_container": graph(
        "unknown_container", [arr("A", ["4"])],
        [{"id": 0, "type": "access", "container": "A"},
         {"id": 1, "type": "tasklet", "name": "t", "ins": ["v"], "outs": ["o"],
          "code": [["o", "v"]]},
         {"id": 2, "type": "access", "container": "A"}],
        [{"src": 0, "dst": 1, "dst_conn": "v", "memlet": "X[0:0:1]"},
         {"src": 1, "dst": 2, "src_conn": "o", "memlet": "A[0:0:1]"}], symbols=()),
    "rank_mismatch": graph(
        "rank_mismatch", [arr("A", ["4", "4"]), arr("x", [], kind="scalar")],
        [{"id": 0, "type": "access", "container": "A"},
         {"id": 1, "type": "tasklet", "name": "t", "ins": ["v"], "outs": ["o"],
          "code": [["o", "v"]]},
         {"id": 2, "type": "access", "container": "x"}],
        [{"src": 0, "dst": 1, "dst_conn": "v", "memlet": "A[0:0:1]"},
         {"src": 1, "dst": 2, "src_conn": "o", "memlet": "x[]"}], symbols=()),
    "sink_not_access": graph(
        "sink_not_access", [arr("x", [], kind="scalar")],
        [{"id": 0, "type": "access", "container": "x"},
         {"id": 1, "type": "tasklet", "name": "t", "ins": ["v"], "outs": ["o"],
          "code": [["o", "v"]]}],
        [{"src": 0, "dst": 1, "dst_conn": "v", "memlet": "x[]"}], symbols=()),
    "unknown_name": graph(
        "unknown_name", [arr("x", [], kind="scalar"), arr("y", [], kind="scalar")],
        [{"id": 0, "type": "access", "container": "x"},
         {"id": 1, "type": "tasklet", "name": "t", "ins": ["v"], "outs": ["o"],
          "code": [["o", "v + q"]]},
         {"id": 2, "type": "access", "container": "y"}],
        [{"src": 0, "dst": 1, "dst_conn": "v", "memlet": "x[]"},
         {"src": 1, "dst": 2, "src_conn": "o", "memlet": "y[]"}], symbols=()),
    "missing_input": graph(
        "missing_input", [arr("x", [], kind="scalar"), arr("y", [], kind="scalar")],
        [{"id": 0, "type": "access", "container": "x"},
         {"id": 1, "type": "tasklet", "name": "t", "ins": ["v", "w"], "outs": ["o"],
          "code": [["o", "v + w"]]},
         {"id": 2, "type": "access", "container": "y"}],
        [{"src": 0, "dst": 1, "dst_conn": "v", "memlet": "x[]"},
         {"src": 1, "dst": 2, "src_conn": "o", "memlet": "y[]"}], symbols=()),
}


def main():
    out = {}
    for name, doc in CASES.items():
        g = serialize.from_dict(json.loads(json.dumps(doc)))
        codes = sorted({d.code for d in g.validate() if d.severity == "error"})
        out[name] = {"graph": doc, "reference_error_codes": codes}
        print(f"{name}: {codes}")
    (HERE / "validation_cases.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
