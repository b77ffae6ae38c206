"""The program-graph IR consumed by the B200 executor.

Input is the reference's serialized graph, JSON schema version 1
(pkg/src/sdfgkit/serialize.py:1-16, 177-282), or a live ``sdfgkit.Sdfg``
object, which is converted through the reference's own ``serialize.to_dict``
(serialize.py:145-174) so both paths see identical data.  The classes here
mirror the reference data model (pkg/src/sdfgkit/ir.py:25-236): containers
with symbolic shapes, access/tasklet/map-entry/map-exit/library/nested nodes,
memlets with inclusive-end strided subsets and optional write-conflict
resolution (WCR), states and interstate transitions.

Node ids are the serialized positions, i.e. the reference's node-id order
(serialize.py:117-119 sorts by nid), so ``State.topological`` reproduces the
reference's deterministic tie-breaking (ir.py:302-322).
"""

from __future__ import annotations

import importlib
import json
from dataclasses import dataclass, field
from typing import Any

from . import scalar, symexpr

SCHEMA_VERSION = 1

DTYPE_BYTES = {"f64": 8, "i64": 8, "i32": 4, "bool": 1}
DTYPE_NP = {"f64": "float64", "i64": "int64", "i32": "int32", "bool": "bool"}
WCR_OPS = ("add", "mul", "min", "max")
COMM_KINDS = {"scatter", "gather", "bcast", "block_scatter", "block_gather",
              "isend", "irecv", "waitall", "dist_matmul"}


class SchemaError(ValueError):
    pass


@dataclass
class Container:
    name: str
    dtype: str
    shape: list  # symexpr trees
    kind: str = "array"  # array | scalar | stream
    transient: bool = False
    lifetime: str = "scope"  # scope | persistent
    storage: str = "heap"  # heap | stack | distributed_local

    @property
    def nbytes_elem(self) -> int:
        return DTYPE_BYTES[self.dtype]


@dataclass
class Memlet:
    container: str
    subset: list  # [(b, e, s)] symexpr trees, inclusive ends
    wcr: str | None = None
    text: str = ""

    def free_symbols(self) -> set[str]:
        out: set[str] = set()
        for d in self.subset:
            for x in d:
                out |= symexpr.free_symbols(x)
        return out


@dataclass(eq=False)
class Node:
    id: int


@dataclass(eq=False)
class Access(Node):
    container: str


@dataclass(eq=False)
class Tasklet(Node):
    name: str
    ins: list
    outs: list
    code: list  # [(out_conn, scalar expr tree)]
    code_text: list = field(default_factory=list)


@dataclass(eq=False)
class MapEntry(Node):
    params: list  # [(name, (b, e, s))]
    schedule: str = "sequential"
    tiled: bool = False

    @property
    def param_names(self) -> list[str]:
        return [p for p, _ in self.params]


@dataclass(eq=False)
class MapExit(Node):
    entry: MapEntry | None = None


@dataclass(eq=False)
class Library(Node):
    kind: str
    name: str
    attrs: dict


@dataclass(eq=False)
class Nested(Node):
    sdfg: "Graph"
    symbol_map: dict  # inner symbol -> symexpr tree (outer names)


@dataclass(eq=False)
class Edge:
    src: Node
    dst: Node
    memlet: Memlet | None
    src_conn: str | None = None
    dst_conn: str | None = None


class State:
    def __init__(self, label: str):
        self.label = label
        self.nodes: list[Node] = []
        self.edges: list[Edge] = []
        self._in: dict[int, list[Edge]] = {}
        self._out: dict[int, list[Edge]] = {}
        self._topo: list[Node] | None = None
        self._parents: dict[int, MapEntry | None] | None = None

    def add(self, n: Node) -> None:
        self.nodes.append(n)
        self._in[n.id] = []
        self._out[n.id] = []

    def add_edge(self, e: Edge) -> None:
        self.edges.append(e)
        self._out[e.src.id].append(e)
        self._in[e.dst.id].append(e)

    def in_edges(self, n: Node) -> list[Edge]:
        return self._in[n.id]

    def out_edges(self, n: Node) -> list[Edge]:
        return self._out[n.id]

    def topological(self) -> list[Node]:
        """Kahn order, ready set sorted by node id (ir.py:302-322)."""
        if self._topo is not None:
            return self._topo
        by_id = {n.id: n for n in self.nodes}
        indeg = {n.id: 0 for n in self.nodes}
        for e in self.edges:
            indeg[e.dst.id] += 1
        ready = sorted(i for i, d in indeg.items() if d == 0)
        order: list[Node] = []
        while ready:
            nid = ready.pop(0)
            order.append(by_id[nid])
            changed = False
            for e in self._out[nid]:
                indeg[e.dst.id] -= 1
                if indeg[e.dst.id] == 0:
                    ready.append(e.dst.id)
                    changed = True
            if changed:
                ready.sort()
        if len(order) != len(self.nodes):
            raise SchemaError(f"cycle in state '{self.label}'")
        self._topo = order
        return order

    def scope_parents(self) -> dict[int, MapEntry | None]:
        """Innermost enclosing map entry of every node (ir.py:324-354)."""
        if self._parents is not None:
            return self._parents
        parent: dict[int, MapEntry | None] = {}
        for node in self.topological():
            preds = self._in[node.id]
            if not preds:
                parent[node.id] = None
                continue
            if isinstance(node, MapExit):
                parent[node.id] = parent[node.entry.id]
                continue
            scopes = set()
            for e in preds:
                s = e.src
                if isinstance(s, MapEntry):
                    scopes.add(s.id)
                elif isinstance(s, MapExit):
                    outer = parent[s.entry.id]
                    scopes.add(outer.id if outer is not None else -1)
                else:
                    p = parent[s.id]
                    scopes.add(p.id if p is not None else -1)
            if len(scopes) != 1:
                raise SchemaError(
                    f"node {node.id} in state '{self.label}' joins different map scopes")
            s = scopes.pop()
            parent[node.id] = None if s == -1 else self.node(s)
        self._parents = parent
        return parent

    def node(self, nid: int) -> Node:
        return self.nodes[nid] if nid < len(self.nodes) and self.nodes[nid].id == nid else \
            next(n for n in self.nodes if n.id == nid)

    def exit_of(self, entry: MapEntry) -> MapExit:
        for n in self.nodes:
            if isinstance(n, MapExit) and n.entry is entry:
                return n
        raise SchemaError(f"map entry {entry.id} has no exit")


@dataclass
class Transition:
    src: str
    dst: str
    condition: Any  # scalar expr tree or None
    assignments: dict  # name -> symexpr tree
    condition_text: str | None = None


class Graph:
    def __init__(self, name: str):
        self.name = name
        self.symbols: dict[str, int] = {}
        self.containers: dict[str, Container] = {}
        self.states: list[State] = []
        self.transitions: list[Transition] = []
        self.start: str | None = None
        self._state_by_label: dict[str, State] = {}
        self._out_tr: dict[str, list[Transition]] = {}
        self.doc: dict | None = None

    def state(self, label: str) -> State:
        return self._state_by_label[label]

    def out_transitions(self, label: str) -> list[Transition]:
        return self._out_tr.get(label, [])

    def free_symbols(self) -> set[str]:
        """Symbols that must be bound by the caller: every name used in
        shapes, memlets, map ranges, tasklets-as-symbols, nested symbol maps and
        transitions that is not a map parameter, container, or assigned by a
        transition (mirrors the role of Sdfg.free_symbols in interp.py:190)."""
        used: set[str] = set()
        for c in self.containers.values():
            for d in c.shape:
                used |= symexpr.free_symbols(d)
        assigned: set[str] = set()
        for t in self.transitions:
            assigned |= set(t.assignments)
            for v in t.assignments.values():
                used |= symexpr.free_symbols(v)
            if t.condition is not None:
                used |= {n for n in scalar.free_names(t.condition) if n not in self.containers}
        for st in self.states:
            parents = st.scope_parents()
            for n in st.nodes:
                if isinstance(n, MapEntry):
                    for _, rng in n.params:
                        for x in rng:
                            used |= symexpr.free_symbols(x)
                elif isinstance(n, Nested):
                    for v in n.symbol_map.values():
                        used |= symexpr.free_symbols(v)
            for e in st.edges:
                if e.memlet is not None:
                    used |= e.memlet.free_symbols()
            _ = parents
        params = set()
        for st in self.states:
            for n in st.nodes:
                if isinstance(n, MapEntry):
                    params |= set(n.param_names)
        return used - params - assigned - set(self.containers)


# ---------------------------------------------------------------------------
# Loading


def _memlet(text: str, wcr: str | None) -> Memlet:
    t = text.strip()
    i = t.find("[")
    if i <= 0 or not t.endswith("]"):
        raise SchemaError(f"bad memlet text {text!r}")
    name = t[:i].strip()
    sub = symexpr.parse_subset(t[i + 1:-1])
    if wcr is not None and wcr not in WCR_OPS:
        raise SchemaError(f"unknown wcr {wcr!r}")
    return Memlet(name, sub, wcr, t)


def _attr(v):
    if isinstance(v, dict):
        if set(v) == {"$expr"}:
            return symexpr.parse(v["$expr"])
        if set(v) == {"$subset"}:
            return symexpr.parse_subset(v["$subset"])
        return {k: _attr(x) for k, x in v.items()}
    if isinstance(v, list):
        return [_attr(x) for x in v]
    return v


def _state(d: dict) -> State:
    st = State(d["label"])
    nodes: list[Node] = []
    pending: list[tuple[MapExit, int]] = []
    for nd in d["nodes"]:
        t = nd["type"]
        nid = nd["id"]
        if t == "access":
            n: Node = Access(nid, nd["container"])
        elif t == "tasklet":
            code = [(c, scalar.parse(x)) for c, x in nd["code"]]
            n = Tasklet(nid, nd.get("name", "t"), list(nd["ins"]), list(nd["outs"]), code,
                        [x for _, x in nd["code"]])
        elif t == "map_entry":
            params = []
            for p, rng in nd["params"]:
                dims = symexpr.parse_subset(rng)
                if len(dims) != 1:
                    raise SchemaError(f"bad map range {rng!r}")
                params.append((p, dims[0]))
            n = MapEntry(nid, params, nd.get("schedule", "sequential"), nd.get("tiled", False))
        elif t == "map_exit":
            n = MapExit(nid, None)
            pending.append((n, nd["entry"]))
        elif t == "library":
            n = Library(nid, nd["kind"], nd.get("name", ""), _attr(nd.get("attrs", {})))
        elif t == "nested":
            n = Nested(nid, from_dict(nd["sdfg"]),
                       {k: symexpr.parse(v) for k, v in nd["symbol_map"].items()})
        else:
            raise SchemaError(f"unknown node type {t!r}")
        st.add(n)
        nodes.append(n)
    by_id = {n.id: n for n in nodes}
    for ex, eid in pending:
        entry = by_id.get(eid)
        if not isinstance(entry, MapEntry):
            raise SchemaError("map_exit does not reference a map_entry")
        ex.entry = entry
    for ed in d["edges"]:
        m = _memlet(ed["memlet"], ed.get("wcr")) if "memlet" in ed else None
        st.add_edge(Edge(by_id[ed["src"]], by_id[ed["dst"]], m,
                         ed.get("src_conn"), ed.get("dst_conn")))
    return st


def from_dict(d: dict) -> Graph:
    if not isinstance(d, dict) or "version" not in d:
        raise SchemaError("not a serialized graph (missing version)")
    if d["version"] != SCHEMA_VERSION:
        raise SchemaError(f"schema version {d['version']} unsupported (want {SCHEMA_VERSION})")
    try:
        g = Graph(d["name"])
        for s in d["symbols"]:
            g.symbols[s["name"]] = s["min"]
        for c in d["containers"]:
            g.containers[c["name"]] = Container(
                c["name"], c["dtype"], [symexpr.parse(s) for s in c["shape"]],
                c.get("kind", "array"), c.get("transient", False),
                c.get("lifetime", "scope"), c.get("storage", "heap"))
        for sd in d["states"]:
            st = _state(sd)
            g.states.append(st)
            g._state_by_label[st.label] = st
        for td in d["transitions"]:
            cond = td.get("condition")
            tr = Transition(td["src"], td["dst"], scalar.parse(cond) if cond else None,
                            {k: symexpr.parse(v) for k, v in td["assignments"].items()}, cond)
            g.transitions.append(tr)
            g._out_tr.setdefault(tr.src, []).append(tr)
        g.start = d["start"]
    except (KeyError, TypeError, IndexError) as ex:
        raise SchemaError(f"malformed graph document: {ex}") from ex
    g.doc = d
    return inline_library_wrappers(g)


WRAPPER_PREFIX = "b200_lib_"


def _wrapped_library(n: Node):
    """The library node held by a b200 expansion wrapper (expansions.py): a
    nested graph named b200_lib_*, one state, one library node whose every
    connector is a whole inner container.  None otherwise."""
    if not isinstance(n, Nested) or not n.sdfg.name.startswith(WRAPPER_PREFIX):
        return None
    inner = n.sdfg
    if len(inner.states) != 1 or inner.transitions:
        return None
    st = inner.states[0]
    libs = [x for x in st.nodes if isinstance(x, Library)]
    if len(libs) != 1 or len(st.nodes) != len(st.edges) + 1:
        return None
    lib = libs[0]
    conn = {}
    for e in st.edges:
        acc = e.src if e.dst is lib else e.dst
        if not isinstance(acc, Access) or e.memlet is None or e.memlet.container != acc.container:
            return None
        from .validate import normalize  # (validate imports this module)

        c = inner.containers[acc.container]
        if len(e.memlet.subset) != len(c.shape):
            return None
        for (b, en, st_), d in zip(e.memlet.subset, c.shape):
            if (normalize(b) != {} or normalize(st_) != {(): 1}
                    or normalize(en) != normalize(("-", d, ("c", 1)))):
                return None
        conn[acc.container] = (e.dst_conn if e.dst is lib else e.src_conn, e.dst is lib)
    if any(symexpr.to_text(v) != k for k, v in n.symbol_map.items()):
        return None
    return lib, conn


def inline_library_wrappers(g: Graph) -> Graph:
    """Put library nodes the b200 registry wrapped (expansions.py) back onto
    their outer memlets, in place: the wrapper's containers are exactly those
    memlets' subsets, so the node reads and writes the same elements (the
    outer write keeps its WCR)."""
    for st in g.states:
        for i, n in enumerate(list(st.nodes)):
            hit = _wrapped_library(n)
            if hit is None:
                continue
            lib, conn = hit
            new = Library(n.id, lib.kind, lib.name, lib.attrs)
            st.nodes[i] = new
            edges = []
            for e in st.edges:
                if e.dst is n:
                    c, _ = conn[e.dst_conn]
                    e = Edge(e.src, new, e.memlet, e.src_conn, c)
                elif e.src is n:
                    c, _ = conn[e.src_conn]
                    e = Edge(new, e.dst, e.memlet, c, e.dst_conn)
                edges.append(e)
            st.edges = []
            st._in = {x.id: [] for x in st.nodes}
            st._out = {x.id: [] for x in st.nodes}
            st._topo = st._parents = None
            for e in edges:
                st.add_edge(e)
        for n in st.nodes:
            if isinstance(n, Nested):
                inline_library_wrappers(n.sdfg)
    return g


def loads(text: str) -> Graph:
    try:
        d = json.loads(text)
    except json.JSONDecodeError as ex:
        raise SchemaError(f"invalid JSON: {ex}") from ex
    return from_dict(d)


def load(path) -> Graph:
    with open(path) as f:
        return loads(f.read())


def as_graph(g) -> Graph:
    """Accept a Graph, a schema-v1 dict/JSON text/path, or an ``sdfgkit.Sdfg``
    (converted with the reference's own serializer, serialize.py:145)."""
    if isinstance(g, Graph):
        return g
    if isinstance(g, dict):
        return from_dict(g)
    if isinstance(g, str):
        s = g.lstrip()
        return loads(g) if s.startswith("{") else load(g)
    if hasattr(g, "states") and hasattr(g, "containers") and hasattr(g, "transitions"):
        root = type(g).__module__.rsplit(".", 1)[0]
        ser = importlib.import_module(root + ".serialize")
        doc = ser.to_dict(g)
        # local-extent symbols of a graph the distribution passes rewrote in
        # place (distribution.py keeps them beside the reference object)
        extra = getattr(g, "_b2_dist_symbols", None)
        if extra:
            doc["dist_symbols"] = dict(extra)
        return from_dict(doc)
    raise TypeError(f"cannot interpret {type(g).__name__} as a program graph")
