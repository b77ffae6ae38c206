"""Graph validation run before execution (unless ``skip_validation``).

Restates the reference's structural validator and static race detector,
``sdfgkit.ir.validate`` (pkg/src/sdfgkit/ir.py:595-745) with
``unordered_hazards`` (ir.py:549-592), ``scope_cross_iteration_hazards``
(ir.py:776-805) / ``_pinned`` (ir.py:762-773), over this package's graph model
(schema v1).  ``Machine.prepare`` raises ``InterpreterError("graph does not
validate: ...")`` on any error diagnostic (interp.py:184-189); so does
``machine.get_executor``.

Disjointness follows ``symbolic.disjoint`` / ``_dim_disjoint``
(symbolic.py:639-692): constant dimensions by point sets, otherwise interval
separation, stride congruence and provable overlap decided on polynomial
normal forms with every declared symbol bounded below by its declared minimum
(``Assumptions``, symbolic.py:211-238; default 1) and unbounded above.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import scalar, sdfg, symexpr

TRUE, FALSE, UNKNOWN = "true", "false", "unknown"
_INF = float("inf")


@dataclass
class Diagnostic:
    severity: str  # "error" | "warning"
    message: str
    code: str
    state: str | None = None
    node: int | None = None


# ---------------------------------------------------------------------------
# polynomial normal form (symbolic.py _normalize / _poly_const)

def _padd(a: dict, b: dict, k: int = 1) -> dict:
    out = dict(a)
    for m, c in b.items():
        v = out.get(m, 0) + k * c
        if v:
            out[m] = v
        else:
            out.pop(m, None)
    return out


def _pmul(a: dict, b: dict) -> dict:
    out: dict = {}
    for ma, ca in a.items():
        for mb, cb in b.items():
            m = tuple(sorted(ma + mb, key=repr))
            v = out.get(m, 0) + ca * cb
            if v:
                out[m] = v
            else:
                out.pop(m, None)
    return out


def normalize(e) -> dict:
    """{monomial (sorted tuple of atoms): integer coefficient}; atoms are
    symbols or opaque floor-div / min / max subtrees (themselves normalised)."""
    tag = e[0]
    if tag == "c":
        return {(): e[1]} if e[1] else {}
    if tag == "s":
        return {(e,): 1}
    if tag == "neg":
        return _padd({}, normalize(e[1]), -1)
    op, l, r = e
    if op == "+":
        return _padd(normalize(l), normalize(r))
    if op == "-":
        return _padd(normalize(l), normalize(r), -1)
    if op == "*":
        return _pmul(normalize(l), normalize(r))
    nl, nr = normalize(l), normalize(r)
    cl, cr = _const(nl), _const(nr)
    if cl is not None and cr is not None:
        v = {"//": lambda a, b: a // b if b else None, "min": min, "max": max}[op](cl, cr)
        if v is not None:
            return {(): v} if v else {}
    atom = (op, _rebuild(nl), _rebuild(nr))
    return {(atom,): 1}


def _const(p: dict):
    if not p:
        return 0
    if set(p) == {()}:
        return p[()]
    return None


def _rebuild(p: dict):
    """A canonical tree for a normal form (used as an opaque atom key)."""
    return ("poly", tuple(sorted(((m, c) for m, c in p.items()), key=repr)))


def _iv_mul(a, b):
    prods = []
    for x in a:
        for y in b:
            if (x == 0 and math.isinf(y)) or (y == 0 and math.isinf(x)):
                prods.append(0.0)
            else:
                prods.append(x * y)
    return (min(prods), max(prods))


def _atom_interval(atom, lower: dict):
    if atom[0] == "s":
        return (float(lower.get(atom[1], 1)), _INF)
    if atom[0] == "poly":
        return _poly_interval(dict(atom[1]), lower)
    op, l, r = atom
    li, ri = _atom_interval(l, lower), _atom_interval(r, lower)
    if op == "min":
        return (min(li[0], ri[0]), min(li[1], ri[1]))
    if op == "max":
        return (max(li[0], ri[0]), max(li[1], ri[1]))
    # floor division: only a positive constant divisor is bounded here
    if ri[0] == ri[1] and ri[0] > 0:
        d = ri[0]
        return (math.floor(li[0] / d) if not math.isinf(li[0]) else li[0],
                math.floor(li[1] / d) if not math.isinf(li[1]) else li[1])
    return (-_INF, _INF)


def _poly_interval(p: dict, lower: dict):
    c0 = float(p.get((), 0))
    lo, hi = c0, c0
    for m, c in p.items():
        if m == ():
            continue
        iv = (1.0, 1.0)
        for a in m:
            iv = _iv_mul(iv, _atom_interval(a, lower))
        iv = _iv_mul(iv, (float(c), float(c)))
        lo, hi = lo + iv[0], hi + iv[1]
    return lo, hi


def compare(lhs: dict, rhs: dict, lower: dict) -> str:
    """``lhs <= rhs`` for every binding within the assumptions (symbolic.py:449)."""
    diff = _padd(lhs, rhs, -1)
    c = _const(diff)
    if c is not None:
        return TRUE if c <= 0 else FALSE
    lo, hi = _poly_interval(diff, lower)
    if hi <= 0:
        return TRUE
    if lo >= 1:
        return FALSE
    return UNKNOWN


def _lt(a: dict, b: dict, lower: dict) -> str:
    return compare(_padd(a, {(): 1}), b, lower)


def _and(*ts):
    if all(t == TRUE for t in ts):
        return TRUE
    if any(t == FALSE for t in ts):
        return FALSE
    return UNKNOWN


def _not(t):
    return {TRUE: FALSE, FALSE: TRUE}.get(t, UNKNOWN)


def dim_disjoint(d1, d2, lower: dict) -> str:
    """symbolic.py:639-678 on normal forms."""
    n1 = [normalize(x) for x in d1]
    n2 = [normalize(x) for x in d2]
    c1 = [_const(x) for x in n1]
    c2 = [_const(x) for x in n2]
    if None not in c1 and None not in c2:
        if c1[2] <= 0 or c2[2] <= 0:
            return TRUE
        p1 = set(range(c1[0], c1[1] + 1, c1[2]))
        p2 = set(range(c2[0], c2[1] + 1, c2[2]))
        return FALSE if p1 & p2 else TRUE
    b1, e1, s1 = n1
    b2, e2, s2 = n2
    ne1, ne2 = compare(b1, e1, lower), compare(b2, e2, lower)
    if _not(ne1) == TRUE or _not(ne2) == TRUE:
        return TRUE
    if _lt(e1, b2, lower) == TRUE or _lt(e2, b1, lower) == TRUE:
        return TRUE
    s1c, s2c, off = _const(s1), _const(s2), _const(_padd(b1, b2, -1))
    if s1c is not None and s2c is not None and off is not None:
        g = math.gcd(s1c, s2c)
        if g > 1 and off % g != 0:
            return TRUE
    if _and(ne1, ne2) == TRUE:
        if b1 == b2:
            return FALSE
        for (pb, pe), (ob, oe, os_) in (((b1, e1), (b2, e2, s2)), ((b2, e2), (b1, e1, s1))):
            if pb == pe:
                inside = _and(compare(ob, pb, lower), compare(pb, oe, lower))
                osc, offp = _const(os_), _const(_padd(pb, ob, -1))
                aligned = TRUE if osc == 1 or (osc is not None and offp is not None
                                               and osc and offp % osc == 0) else UNKNOWN
                if _and(inside, aligned) == TRUE:
                    return FALSE
    return UNKNOWN


def disjoint(s1: list, s2: list, lower: dict) -> str:
    if len(s1) != len(s2):
        raise ValueError(f"rank mismatch: {len(s1)} vs {len(s2)}")
    if not s1:
        return FALSE  # two scalars always collide
    per = [dim_disjoint(a, b, lower) for a, b in zip(s1, s2)]
    if any(v == TRUE for v in per):
        return TRUE
    if all(v == FALSE for v in per):
        return FALSE
    return UNKNOWN


# ---------------------------------------------------------------------------
# hazards


def _reachability(st: sdfg.State) -> dict:
    reach = {n.id: set() for n in st.nodes}
    for n in reversed(st.topological()):
        for e in st.out_edges(n):
            reach[n.id].add(e.dst.id)
            reach[n.id] |= reach[e.dst.id]
    return reach


def unordered_hazards(st: sdfg.State, lower: dict) -> list:
    """ir.py:549-592: same-container access pairs with a write and no path."""
    reach = _reachability(st)
    by: dict = {}
    for n in st.topological():
        if isinstance(n, sdfg.Access):
            by.setdefault(n.container, []).append(n)
    out = []
    for cont, occs in by.items():
        for i in range(len(occs)):
            for j in range(i + 1, len(occs)):
                u, v = occs[i], occs[j]
                if v.id in reach[u.id] or u.id in reach[v.id]:
                    continue
                uw = [e.memlet for e in st.in_edges(u) if e.memlet is not None]
                ur = [e.memlet for e in st.out_edges(u) if e.memlet is not None]
                vw = [e.memlet for e in st.in_edges(v) if e.memlet is not None]
                vr = [e.memlet for e in st.out_edges(v) if e.memlet is not None]
                if not uw and not vw:
                    continue
                verdicts = []
                for m1, others in ((uw, vw + vr), (vw, ur)):
                    for a in m1:
                        for b in others:
                            if a.wcr is not None and b.wcr == a.wcr:
                                continue  # commuting conflict resolution
                            verdicts.append(disjoint(a.subset, b.subset, lower))
                if not verdicts:
                    continue
                verdict = _and(*verdicts) if all(x != FALSE for x in verdicts) else FALSE
                if verdict != TRUE:
                    out.append((cont, u, v, verdict))
    return out


def _pinned(param: str, params: set, w: list, x: list) -> bool:
    """ir.py:762-773."""
    for (wb, we, _), (xb, xe, _) in zip(w, x):
        if normalize(wb) != normalize(we) or normalize(xb) != normalize(xe):
            continue
        if normalize(wb) != normalize(xb):
            continue
        if symexpr.free_symbols(wb) & params == {param}:
            return True
    return False


def cross_iteration_hazards(st: sdfg.State, entry: sdfg.MapEntry) -> list:
    """ir.py:776-805: boundary memlets that may collide across iterations."""
    ex = next(n for n in st.nodes if isinstance(n, sdfg.MapExit) and n.entry is entry)
    reads: dict = {}
    writes: dict = {}
    for e in st.out_edges(entry):
        if e.memlet is not None:
            reads.setdefault(e.memlet.container, []).append(e.memlet)
    for e in st.in_edges(ex):
        if e.memlet is not None:
            writes.setdefault(e.memlet.container, []).append(e.memlet)
    params = set(entry.param_names)
    out = []
    for cont, wl in writes.items():
        for w in wl:
            for x in wl + reads.get(cont, []):
                if w.wcr is not None and x.wcr == w.wcr:
                    continue
                if all(_pinned(p, params, w.subset, x.subset) for p in params):
                    continue
                out.append((cont, w, x))
    return out


# ---------------------------------------------------------------------------


def _assigned(g: sdfg.Graph) -> set:
    out: set = set()
    for t in g.transitions:
        out |= set(t.assignments)
    return out


def validate(g: sdfg.Graph) -> list[Diagnostic]:
    """ir.py:595-745 restated; returns diagnostics instead of raising."""
    diags: list[Diagnostic] = []

    def err(msg, code, state=None, node=None):
        diags.append(Diagnostic("error", msg, code, state, node))

    labels = [s.label for s in g.states]
    if g.start is None or g.start not in labels:
        err(f"missing or unknown start state '{g.start}'", "start-state")
        return diags
    if len(set(labels)) != len(labels):
        err("duplicate state labels", "state-labels")
    lower = dict(g.symbols)
    known = set(g.containers) | set(g.symbols) | _assigned(g)
    for c in g.containers.values():
        for d in c.shape:
            for s in symexpr.free_symbols(d):
                if s not in g.symbols:
                    err(f"shape of '{c.name}' uses undeclared symbol '{s}'", "unknown-symbol")
        if c.kind == "scalar" and c.shape:
            err(f"scalar '{c.name}' has a shape", "scalar-shape")
        if c.kind == "stream" and len(c.shape) != 1:
            err(f"stream '{c.name}' must be one-dimensional", "stream-rank")
    for st in g.states:
        try:
            st.topological()
        except (ValueError, sdfg.SchemaError) as ex:
            err(str(ex), "state-cycle", st.label)
            continue
        try:
            parents = st.scope_parents()
        except (ValueError, sdfg.SchemaError) as ex:
            err(str(ex), "scope-structure", st.label)
            continue
        entries = [n for n in st.nodes if isinstance(n, sdfg.MapEntry)]
        exits = [n for n in st.nodes if isinstance(n, sdfg.MapExit)]
        if len(entries) != len(exits) or {id(x.entry) for x in exits} != {id(e) for e in entries}:
            err("unbalanced map entry/exit pairs", "scope-brackets", st.label)

        def scope_params(n):
            out = set()
            cur = parents.get(n.id)
            while cur is not None:
                out |= set(cur.param_names)
                cur = parents.get(cur.id)
            return out

        for e in st.edges:
            m = e.memlet
            if m is None:
                continue
            c = g.containers.get(m.container)
            if c is None:
                err(f"unknown container {m.container}", "unknown-container", st.label)
                continue
            if len(m.subset) != len(c.shape):
                err(f"memlet {m.text} has rank {len(m.subset)}, container has rank "
                    f"{len(c.shape)}", "rank-mismatch", st.label)
            if m.wcr is not None and not isinstance(e.dst, (sdfg.Access, sdfg.MapExit)):
                err(f"wcr memlet {m.text} on a non-write edge", "wcr-read", st.label, e.dst.id)
            pnames = set()
            if isinstance(e.src, sdfg.MapEntry):
                pnames |= set(e.src.param_names)
            if isinstance(e.dst, sdfg.MapExit) and e.dst.entry is not None:
                pnames |= set(e.dst.entry.param_names)
            pnames |= scope_params(e.src) | scope_params(e.dst)
            for s in m.free_symbols():
                if s not in known and s not in pnames:
                    err(f"memlet {m.text} uses undeclared name '{s}'", "unknown-symbol", st.label)
        for n in st.nodes:
            if not st.out_edges(n) and not isinstance(n, sdfg.Access):
                err(f"{type(n).__name__} {n.id} is a dataflow sink", "sink-not-access",
                    st.label, n.id)
            if isinstance(n, sdfg.Tasklet):
                conns = {e.dst_conn for e in st.in_edges(n)}
                missing = set(n.ins) - conns
                if missing:
                    err(f"tasklet {n.name} missing inputs {sorted(missing)}", "missing-input",
                        st.label, n.id)
                sp = scope_params(n)
                for _, code in n.code:
                    for name in scalar.free_names(code):
                        if name not in n.ins and name not in known and name not in sp:
                            err(f"tasklet {n.name} references unknown name '{name}'",
                                "unknown-name", st.label, n.id)
        for cont, u, _v, verdict in unordered_hazards(st, lower):
            if verdict == FALSE:
                err(f"data race on {cont}", "data-race", st.label, u.id)
            else:
                err(f"possible data race on {cont} (unprovable disjointness)", "data-race",
                    st.label, u.id)
        for entry in entries:
            if entry.schedule == "sequential":
                continue
            if not any(isinstance(x, sdfg.MapExit) and x.entry is entry for x in st.nodes):
                continue
            for cont, _w, _x in cross_iteration_hazards(st, entry):
                err(f"data race on {cont}", "data-race", st.label, entry.id)
    for t in g.transitions:
        if t.src not in labels or t.dst not in labels:
            err(f"transition {t.src}->{t.dst} references unknown state", "unknown-state")
            continue
        if t.condition is not None:
            for name in scalar.free_names(t.condition):
                if name not in known:
                    err(f"condition on {t.src}->{t.dst} uses undeclared name '{name}'",
                        "unknown-symbol")
    return diags


def errors(g: sdfg.Graph) -> list[Diagnostic]:
    return [d for d in validate(g) if d.severity == "error"]
