"""The B200 library plug-in for the reference's expansion registry.

The reference expands library nodes through a per-kind priority list
(``ExpansionRegistry`` / ``Expansion(name, applicable, apply)``,
pkg/src/sdfgkit/autoopt.py:640-664) driven by ``expand_library``
(autoopt.py:958-983), which ``auto_optimize`` calls last (autoopt.py:990).
Its CPU entries rewrite MATMUL / REDUCE / TRANSPOSE into WCR maps
(``_expand_matmul_native`` 707-813, ``_expand_reduce_native`` 816-876), which
is the right thing for a Python interpreter and the wrong one for a B200:
those nodes have device library kernels here (rowpass BLAS-2 family, DMMA
DGEMM, b2_reduce, b2_copy_view).

``B200_EXPANSIONS`` are registry entries named ``"b200"`` that keep such a
node as a device library node.  ``expand_library`` keeps looping while any
top-level MATMUL / REDUCE / TRANSPOSE node remains (autoopt.py:969-981), so
the expansion moves the node one level down: into a single-state nested
graph whose containers are exactly the node's memlet subsets (connector ==
inner container, the outer memlets keep their WCR, interp.py:491-517).  The
reference interpreter runs that wrapper with unchanged semantics; this
backend's loader (``sdfg.inline_library_wrappers``) puts the node back onto
the outer memlets, so the device kernels — including the BLAS-2 fusions
across adjacent products — see it as if it had never been expanded.

Use:
  * ``b200_registry(base)`` — a registry with the b200 entries ahead of
    ``base``'s (e.g. ``autoopt.cpu_registry()``), for
    ``expand_library(g, registry=..., pinned=...)``;
  * ``install(reg)`` — prepend them to an existing reference registry;
  * ``patched_cpu_registry(autoopt)`` — context manager that makes
    ``autoopt.cpu_registry()`` (hence ``auto_optimize``) return such a
    registry.
"""

from __future__ import annotations

import contextlib
import importlib
from dataclasses import dataclass
from typing import Callable

WRAPPER_PREFIX = "b200_lib_"
KINDS = ("matmul", "reduce", "transpose")
_REDUCE_OPS = ("add", "mul", "min", "max")
_DTYPES = ("f64",)  # the device library kernels' element type


@dataclass
class Expansion:
    """Duck-typed twin of autoopt.Expansion (name, applicable, apply)."""

    name: str
    applicable: Callable
    apply: Callable


def _ref(g):
    root = type(g).__module__.rsplit(".", 1)[0]
    return importlib.import_module(root + ".ir"), importlib.import_module(root + ".symbolic")


def _dtype_ok(g, st, node) -> bool:
    for e in list(st.in_edges(node)) + list(st.out_edges(node)):
        if e.memlet is None:
            continue
        d = g.containers.get(e.memlet.container)
        if d is None or d.dtype.value not in _DTYPES:
            return False
    return True


def _applicable(g, st, node) -> bool:
    kind = node.kind.value
    if kind not in KINDS or not _dtype_ok(g, st, node):
        return False
    ins = [e for e in st.in_edges(node) if e.memlet is not None]
    outs = [e for e in st.out_edges(node) if e.memlet is not None]
    if len(outs) != 1:
        return False
    if kind == "matmul":
        conns = {e.dst_conn for e in ins}
        if conns != {"a", "b"}:
            return False
        # inner-dimension mismatches stay with the native expansion, which
        # raises the reference's ValueError("inner dimensions ...")
        try:
            importlib.import_module(type(g).__module__.rsplit(".", 1)[0] + ".autoopt") \
                ._matmul_dims(g, st, node)
        except Exception:  # noqa: BLE001
            return False
        return True
    if kind == "reduce":
        return len(ins) == 1 and node.attributes.get("op", "add") in _REDUCE_OPS
    return len(ins) == 1  # transpose


def _extent(sym, b, e, s):
    return sym.simplify(sym.Add(sym.FloorDiv(sym.Sub(e, b), s), sym.Const(1)))


def _wrap(g, st, node) -> None:
    """Replace ``node`` by a single-state nested graph that holds it."""
    ir, sym = _ref(g)
    inner = ir.Sdfg(f"{WRAPPER_PREFIX}{node.kind.value}_{node.nid}")
    ist = inner.add_state("s0", start=True)
    lib = ist.add(ir.LibraryNode(node.kind, node.name, dict(node.attributes)))
    outer_edges = []
    used = set()
    for e in list(st.in_edges(node)) + list(st.out_edges(node)):
        if e.memlet is None:
            continue
        incoming = e.dst is node
        conn = e.dst_conn if incoming else e.src_conn
        cname = conn if conn not in used else f"{conn}_{len(used)}"
        used.add(cname)
        desc = g.containers[e.memlet.container]
        shape = tuple(_extent(sym, b, en, s) for (b, en, s) in e.memlet.subset.dims)
        for d in shape:
            for s_ in d.free_symbols():
                inner.add_symbol(s_, g.symbols.get(s_, 1))
        # outputs are scratch inside the wrapper: the outer memlet (and its
        # WCR) writes them back (interp.py:511-516)
        transient = not incoming
        if desc.kind is ir.DataKind.SCALAR:
            inner.add_scalar(cname, desc.dtype, transient=transient)
            full = sym.SubsetRange(())
        else:
            inner.add_array(cname, desc.dtype, shape, transient=transient)
            full = sym.SubsetRange.full(shape)
        acc = ist.add(ir.AccessNode(cname))
        if incoming:
            ist.add_edge(acc, lib, ir.Memlet(cname, full), dst_conn=conn)
        else:
            ist.add_edge(lib, acc, ir.Memlet(cname, full), src_conn=conn)
        outer_edges.append((e, cname, incoming))
    symbol_map = {s_: sym.Sym(s_) for s_ in inner.symbols}
    nested = st.add(ir.NestedSdfg(inner, symbol_map))
    for e, cname, incoming in outer_edges:
        if incoming:
            st.add_edge(e.src, nested, e.memlet, src_conn=e.src_conn, dst_conn=cname)
        else:
            st.add_edge(nested, e.dst, e.memlet, src_conn=cname, dst_conn=e.dst_conn)
    st.remove_node(node)


B200_EXPANSIONS = {k: Expansion("b200", _applicable, _wrap) for k in KINDS}


class Registry:
    """Duck-typed ExpansionRegistry (by_kind / register / pick) keyed by the
    kind's value, so it needs no import of the reference."""

    def __init__(self):
        self.by_kind: dict = {}

    def register(self, kind, expansion) -> None:
        self.by_kind.setdefault(getattr(kind, "value", kind), []).append(expansion)

    def pick(self, g, st, node, pinned=None):
        cands = self.by_kind.get(node.kind.value, [])
        if pinned and node.kind.value in pinned:
            cands = [x for x in cands if x.name == pinned[node.kind.value]]
        for x in cands:
            if x.applicable(g, st, node):
                return x
        return None


def b200_registry(base=None) -> Registry:
    """b200 entries first, then ``base``'s entries (kind by kind)."""
    reg = Registry()
    for k, x in B200_EXPANSIONS.items():
        reg.register(k, x)
    if base is not None:
        for kind, lst in base.by_kind.items():
            for x in lst:
                reg.register(kind, x)
    return reg


def install(reg) -> None:
    """Prepend the b200 entries to a reference ``ExpansionRegistry``."""
    kinds = {k.value: k for k in reg.by_kind}
    for k, x in B200_EXPANSIONS.items():
        if k in kinds:
            reg.by_kind[kinds[k]].insert(0, x)


@contextlib.contextmanager
def patched_cpu_registry(autoopt):
    """``autoopt.cpu_registry()`` (used by ``expand_library`` / ``auto_optimize``
    when no registry is given) returns the b200-first registry inside."""
    orig = autoopt.cpu_registry

    def reg():
        r = orig()
        install(r)
        return r

    autoopt.cpu_registry = reg
    try:
        yield
    finally:
        autoopt.cpu_registry = orig
