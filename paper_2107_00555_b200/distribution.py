"""Global-view distribution passes (the reference's missing ``sdfgkit.dist``
transformations, restated from SPEC.md:544-571 and the behaviour
pkg/tests/test_dist.py pins), on schema-v1 graph documents.

* ``distribute_elementwise`` (paper Fig. 7): a top-level
  parallel map whose every memlet indexes dimension d of its container with
  ``param_d + const`` is rewritten to: Bcast of the scalars it reads,
  BlockScatter (2-D grids: block rows x block columns of the map's first two
  dimensions; 1-D maps: flat Scatter of a dense view, else rows) of every
  input view into a DISTRIBUTED_LOCAL transient, the map re-ranged to the
  local extents, BlockGather / Gather of every output view, and a Reduce
  (the memlet's WCR operator, result at the root) for a WCR output of rank 0.
* ``expand_matmul_distributed``: a 2D@2D MATMUL of whole
  2-D views becomes BlockScatter(A), BlockScatter(B), DIST_MATMUL (SUMMA over
  K panels: row broadcast of the A panel, column broadcast of the B panel,
  comm.RankComm._dist_matmul) and BlockGather(C).
* ``remove_redundant_comm`` (paper §4.2 / Fig. 9): a
  Gather / BlockGather of local X into global transient T whose only reader
  is a Scatter / BlockScatter back into local X' with the same distribution
  (grid, scheme, block, global extents) is removed; X' is replaced by X.
* ``distribution_pipeline`` = distribute + remove_redundant_comm.

Operations the passes do not distribute (REDUCE / TRANSPOSE / matrix-vector
products, loops of scalar code, maps with shifted-by-parameter indexing)
stay global: they run on the root rank only (the reference's
``dist_nonroot`` root-resident containers, interp.py:165-170, 199-206).

Local extents are symbols ``__dl<k>`` recorded in the document under
``"dist_symbols"`` ({symbol: {"extent": global extent text, "dim": grid
dimension or null, "grid": [...], "block": text}}); ``local_bindings``
evaluates them per rank.  Block extents that the grid does not divide are a
hard error ("no implicit padding").
"""

from __future__ import annotations

import copy
import importlib
import json
import math

from . import sdfg, symexpr

COLLECTIVES = ("scatter", "gather", "bcast", "block_scatter", "block_gather")


class DistError(ValueError):
    pass


def _dims(grid) -> list:
    d = list(getattr(grid, "dims", grid))
    if not d or len(d) > 2 or any(int(x) < 1 for x in d):
        raise DistError(f"bad process grid {d}")
    return [int(x) for x in d]


def _coords(dims, r):
    return (r // dims[1], r % dims[1]) if len(dims) == 2 else (r,)


# ---------------------------------------------------------------------------
# document helpers


def _parse_memlet(text):
    t = text.strip()
    i = t.index("[")
    return t[:i].strip(), symexpr.parse_subset(t[i + 1:-1])


def _memlet(cont, dims):
    return f"{cont}[" + ", ".join(
        f"{symexpr.to_text(b)}:{symexpr.to_text(e)}:{symexpr.to_text(s)}" for b, e, s in dims) + "]"


def _const(e):
    try:
        return symexpr.evaluate(e, {})
    except KeyError:
        return None


class _Doc:
    def __init__(self, doc):
        self.d = doc
        self.cont = {c["name"]: c for c in doc["containers"]}
        self.dsym = doc.setdefault("dist_symbols", {})
        self.report: dict = {}

    def count(self, key, n=1):
        self.report[key] = self.report.get(key, 0) + n

    def fresh_cont(self, base, dtype, shape, kind="array"):
        k = 0
        while f"{base}{k}" in self.cont:
            k += 1
        name = f"{base}{k}"
        c = {"name": name, "dtype": dtype, "shape": shape, "kind": kind, "transient": True,
             "lifetime": "scope", "storage": "distributed_local"}
        self.d["containers"].append(c)
        self.cont[name] = c
        return name

    def fresh_sym(self, extent_text, dim, grid, block=None):
        k = len(self.dsym)
        while f"__dl{k}" in self.dsym:
            k += 1
        name = f"__dl{k}"
        self.dsym[name] = {"extent": extent_text, "dim": dim, "grid": list(grid),
                           "block": block}
        self.d["symbols"].append({"name": name, "min": 1})
        return name


def _next_id(st):
    return max([n["id"] for n in st["nodes"]], default=-1) + 1


def _scope_nodes(st, entry_id):
    """Ids of the nodes strictly inside a top-level map scope."""
    by = {n["id"]: n for n in st["nodes"]}
    exit_id = next(n["id"] for n in st["nodes"] if n["type"] == "map_exit"
                   and n["entry"] == entry_id)
    inside, stack = set(), [entry_id]
    while stack:
        cur = stack.pop()
        for e in st["edges"]:
            if e["src"] == cur and e["dst"] not in inside and e["dst"] != exit_id:
                inside.add(e["dst"])
                stack.append(e["dst"])
    return inside, exit_id, by


def _top_level_entries(st):
    entries = [n for n in st["nodes"] if n["type"] == "map_entry"]
    inner = set()
    for n in entries:
        ins, _, _ = _scope_nodes(st, n["id"])
        inner |= ins
    return [n for n in entries if n["id"] not in inner]


# ---------------------------------------------------------------------------
# distribute_elementwise


def _elementwise_plan(D: _Doc, st, entry):
    """(params, ranges, boundary info) when the map is element-wise, else None."""
    if entry.get("schedule") != "parallel":
        return None
    params = [p for p, _ in entry["params"]]
    ranges = [symexpr.parse_subset(r)[0] for _, r in entry["params"]]
    if any(_const(s) != 1 for _, _, s in ranges):
        return None
    inside, exit_id, by = _scope_nodes(st, entry["id"])
    if any(by[i]["type"] in ("map_entry", "library", "nested") for i in inside):
        return None
    k = len(params)
    views = {}  # (cont, offsets, is_write, wcr) -> list of inner edge indices
    for idx, e in enumerate(st["edges"]):
        if "memlet" not in e:
            continue
        inner_edge = (e["src"] == entry["id"] and e["dst"] in inside) or \
                     (e["dst"] == exit_id and e["src"] in inside)
        if not inner_edge:
            continue
        cont, sub = _parse_memlet(e["memlet"])
        c = D.cont.get(cont)
        if c is None or c.get("storage") == "distributed_local":
            return None
        write = e["dst"] == exit_id
        if c["kind"] == "scalar" or not sub:
            # a rank-0 output must be a WCR add: ranks accumulate from the
            # local transient's zeros and a Reduce combines them at the root
            if write and e.get("wcr") != "add":
                return None
            views.setdefault((cont, (), write, e.get("wcr") if write else None), []).append(idx)
            continue
        if len(sub) != k or write and e.get("wcr"):
            return None
        offs = []
        for d, (b, en, s) in enumerate(sub):
            if symexpr.to_text(b) != symexpr.to_text(en):
                return None
            a = symexpr.affine(b, tuple(params), {})
            if a is None:
                return None
            c0, co = a
            if dict(co) != {params[d]: 1} or not isinstance(c0, int):
                return None
            offs.append(c0)
        views.setdefault((cont, tuple(offs), write, None), []).append(idx)
    if not views or not any(w for (_, _, w, _) in views):
        return None
    return params, ranges, views, inside, exit_id


def _extent_text(rng):
    b, e, _ = rng
    return symexpr.to_text(symexpr.parse(f"({symexpr.to_text(e)}) - ({symexpr.to_text(b)}) + 1"))


def distribute_elementwise(doc: dict, grid, blocks=None) -> dict:
    """Distribute every element-wise top-level map (see module doc)."""
    D = _Doc(doc)
    dims = _dims(grid)
    P = math.prod(dims)
    for st in doc["states"]:
        for entry in list(_top_level_entries(st)):
            plan = _elementwise_plan(D, st, entry)
            if plan is None:
                continue
            _distribute_map(D, st, entry, plan, dims, P)
            D.count("distribute_elementwise")
    return D.report


def _distribute_map(D: _Doc, st, entry, plan, dims, P):
    params, ranges, views, inside, exit_id = plan
    k = len(params)
    ext = [_extent_text(r) for r in ranges]
    # distribution of the iteration space: 2-D grids split the first two
    # map dims (block rows x block columns), 1-D grids the first one
    gdims = dims if len(dims) == 2 else [dims[0]]
    if k == 1:
        gdims = [P]
    scheme_grid = gdims[: min(len(gdims), k)]
    lsym = []
    for d in range(k):
        if d < len(scheme_grid):
            lsym.append(D.fresh_sym(ext[d], d, scheme_grid))
        else:
            lsym.append(None)
    lshape = [s if s is not None else ext[d] for d, s in enumerate(lsym)]
    nid = _next_id(st)
    new_nodes, new_edges = [], []
    dist_attr = {"grid": list(scheme_grid), "block": [
        f"({e}) // {g}" for e, g in zip(ext, scheme_grid)], "scheme": "block"}
    local_of = {}
    for (cont, offs, write, wcr), idxs in sorted(views.items(), key=lambda kv: str(kv[0])):
        c = D.cont[cont]
        if not offs:  # scalar
            lname = D.fresh_cont("__dls", c["dtype"], [], "scalar")
            gm, lm = f"{cont}[]", f"{lname}[]"
        else:
            lname = D.fresh_cont("__dla", c["dtype"], list(lshape))
            gdims_ = [(symexpr.parse(f"({symexpr.to_text(ranges[d][0])}) + {offs[d]}"),
                       symexpr.parse(f"({symexpr.to_text(ranges[d][1])}) + {offs[d]}"),
                       ("c", 1)) for d in range(k)]
            gm = _memlet(cont, gdims_)
            lm = _memlet(lname, [(("c", 0), symexpr.parse(f"({s}) - 1"), ("c", 1))
                                 for s in lshape])
        local_of[(cont, offs, write, wcr)] = lname
        g_acc = {"id": nid, "type": "access", "container": cont}
        l_acc = {"id": nid + 1, "type": "access", "container": lname}
        if not offs:
            kind = "reduce" if write else "bcast"
        elif k == 1 and len(dims) >= 1:
            kind = ("gather" if write else "scatter") if _dense_1d(D, cont, gdims_) else \
                ("block_gather" if write else "block_scatter")
        else:
            kind = "block_gather" if write else "block_scatter"
        attrs = {"dist": dist_attr} if kind.startswith("block") else {}
        if kind == "reduce":
            attrs = {"op": wcr, "comm": True}
        lib = {"id": nid + 2, "type": "library", "kind": kind, "name": kind, "attrs": attrs}
        new_nodes += [g_acc, l_acc, lib]
        if write:  # local -> collective -> global
            e1 = {"src": l_acc["id"], "dst": lib["id"], "dst_conn": "a", "memlet": lm}
            e2 = {"src": lib["id"], "dst": g_acc["id"], "src_conn": "out", "memlet": gm}
            if kind == "reduce":
                e2["wcr"] = wcr
            new_edges += [e1, e2]
            D.count(f"insert_{kind}")
        else:  # global -> collective -> local
            new_edges += [{"src": g_acc["id"], "dst": lib["id"], "dst_conn": "a", "memlet": gm},
                          {"src": lib["id"], "dst": l_acc["id"], "src_conn": "out", "memlet": lm}]
            D.count(f"insert_{kind}")
        nid += 3
    # re-range the map and point its memlets at the local transients
    entry["params"] = [[p, f"0:({lshape[d]}) - 1:1"] for d, p in enumerate(params)]
    for (cont, offs, write, wcr), idxs in views.items():
        lname = local_of[(cont, offs, write, wcr)]
        for i in idxs:
            e = st["edges"][i]
            if not offs:
                e["memlet"] = f"{lname}[]"
            else:
                e["memlet"] = _memlet(lname, [(("s", p), ("s", p), ("c", 1)) for p in params])
    # boundary edges: outside access nodes <-> entry / exit become local ones
    lacc_id = {}
    for n in new_nodes:
        if n["type"] == "access" and n["container"] in D.cont and \
                D.cont[n["container"]].get("storage") == "distributed_local":
            lacc_id[n["container"]] = n["id"]
    keep = []
    outside_acc = set()
    for e in st["edges"]:
        if e["dst"] == entry["id"] and "memlet" in e:
            outside_acc.add(e["src"])
            continue  # replaced below
        if e["src"] == exit_id and "memlet" in e:
            outside_acc.add(e["dst"])
            continue
        keep.append(e)
    st["edges"] = keep
    for (cont, offs, write, wcr) in views:
        lname = local_of[(cont, offs, write, wcr)]
        full = (f"{lname}[]" if not offs else
                _memlet(lname, [(("c", 0), symexpr.parse(f"({s}) - 1"), ("c", 1)) for s in lshape]))
        if write:
            st["edges"].append({"src": exit_id, "dst": lacc_id[lname], "src_conn": f"OUT_{lname}",
                                "memlet": full, **({"wcr": wcr} if wcr else {})})
            for e in st["edges"]:
                if e.get("dst") == exit_id and e.get("memlet", "").startswith(lname + "["):
                    e["dst_conn"] = f"IN_{lname}"
        else:
            st["edges"].append({"src": lacc_id[lname], "dst": entry["id"],
                                "dst_conn": f"IN_{lname}", "memlet": full})
            for e in st["edges"]:
                if e.get("src") == entry["id"] and e.get("memlet", "").startswith(lname + "["):
                    e["src_conn"] = f"OUT_{lname}"
    st["nodes"] += new_nodes
    st["edges"] += new_edges
    # outside access nodes that lost all their edges
    used = {e["src"] for e in st["edges"]} | {e["dst"] for e in st["edges"]}
    st["nodes"] = [n for n in st["nodes"] if n["id"] in used or n["id"] not in outside_acc]


def _dense_1d(D, cont, dims_):
    c = D.cont[cont]
    if len(c["shape"]) != 1:
        return False
    b, e, _ = dims_[0]
    return _const(b) == 0 and _norm(symexpr.parse(f"({symexpr.to_text(e)}) + 1")) == \
        _norm(symexpr.parse(c["shape"][0]))


# ---------------------------------------------------------------------------
# expand_matmul_distributed


def expand_matmul_distributed(doc: dict, grid) -> dict:
    D = _Doc(doc)
    dims = _dims(grid)
    g2 = dims if len(dims) == 2 else [dims[0], 1]
    for st in doc["states"]:
        for n in list(st["nodes"]):
            if n["type"] != "library" or n["kind"] != "matmul":
                continue
            ins = {e["dst_conn"]: e for e in st["edges"] if e["dst"] == n["id"] and "memlet" in e}
            outs = [e for e in st["edges"] if e["src"] == n["id"] and "memlet" in e]
            if set(ins) != {"a", "b"} or len(outs) != 1 or outs[0].get("wcr"):
                continue
            views = []
            for e in (ins["a"], ins["b"], outs[0]):
                cont, sub = _parse_memlet(e["memlet"])
                if len(sub) != 2 or any(_const(s) != 1 for _, _, s in sub):
                    break
                views.append((cont, sub))
            if len(views) != 3 or any(not all(n["attrs"].get(k, [True, True]))
                                      for k in ("a_kept", "b_kept")):
                continue
            (ca, sa), (cb, sb), (cc, sc) = views
            ea = [_extent_text(r) for r in sa]
            eb = [_extent_text(r) for r in sb]
            ec = [_extent_text(r) for r in sc]
            nid = _next_id(st)
            new_nodes, new_edges, loc = [], [], {}
            for role, cont, sub, ex in (("a", ca, sa, ea), ("b", cb, sb, eb), ("c", cc, sc, ec)):
                s0 = D.fresh_sym(ex[0], 0, g2)
                s1 = D.fresh_sym(ex[1], 1, g2)
                lname = D.fresh_cont("__dlm", D.cont[cont]["dtype"], [s0, s1])
                loc[role] = (lname, f"{lname}[0:({s0}) - 1:1, 0:({s1}) - 1:1]", ex)
            dist_for = {r: {"grid": list(g2), "block": [f"({x[2][0]}) // {g2[0]}",
                                                         f"({x[2][1]}) // {g2[1]}"],
                            "scheme": "block"} for r, x in loc.items()}
            # global operand -> BlockScatter -> local
            for role, e in (("a", ins["a"]), ("b", ins["b"])):
                lname, lm, _ = loc[role]
                la = {"id": nid, "type": "access", "container": lname}
                sc_ = {"id": nid + 1, "type": "library", "kind": "block_scatter",
                       "name": "block_scatter", "attrs": {"dist": dist_for[role]}}
                new_nodes += [la, sc_]
                new_edges += [{"src": e["src"], "dst": sc_["id"], "dst_conn": "a",
                               "memlet": e["memlet"]},
                              {"src": sc_["id"], "dst": la["id"], "src_conn": "out",
                               "memlet": lm}]
                loc[role] = (lname, lm, la["id"])
                nid += 2
                D.count("insert_block_scatter")
            lname, lm, _ = loc["c"]
            lc = {"id": nid, "type": "access", "container": lname}
            dm = {"id": nid + 1, "type": "library", "kind": "dist_matmul", "name": "dist_matmul",
                  "attrs": {"dist": dist_for["c"]}}
            ga = {"id": nid + 2, "type": "library", "kind": "block_gather",
                  "name": "block_gather", "attrs": {"dist": dist_for["c"]}}
            new_nodes += [lc, dm, ga]
            new_edges += [{"src": loc["a"][2], "dst": dm["id"], "dst_conn": "a",
                           "memlet": loc["a"][1]},
                          {"src": loc["b"][2], "dst": dm["id"], "dst_conn": "b",
                           "memlet": loc["b"][1]},
                          {"src": dm["id"], "dst": lc["id"], "src_conn": "out", "memlet": lm},
                          {"src": lc["id"], "dst": ga["id"], "dst_conn": "a", "memlet": lm},
                          {"src": ga["id"], "dst": outs[0]["dst"], "src_conn": "out",
                           "memlet": outs[0]["memlet"]}]
            st["edges"] = [e for e in st["edges"] if e["src"] != n["id"] and e["dst"] != n["id"]]
            st["nodes"] = [x for x in st["nodes"] if x["id"] != n["id"]]
            st["nodes"] += new_nodes
            st["edges"] += new_edges
            D.count("expand_matmul_distributed")
            D.count("insert_block_gather")
    return D.report


# ---------------------------------------------------------------------------
# remove_redundant_comm


def _chain_states(doc, a, b):
    """True when state b follows state a through unconditional single
    transitions (a straight line), or a == b."""
    if a == b:
        return True
    outs = {}
    for t in doc["transitions"]:
        outs.setdefault(t["src"], []).append(t)
    cur, seen = a, set()
    while cur not in seen:
        seen.add(cur)
        ts = outs.get(cur, [])
        if len(ts) != 1 or ts[0].get("condition"):
            return False
        cur = ts[0]["dst"]
        if cur == b:
            return True
    return False


def _same_dist(D, x_local, xp_local, gat, sca):
    if gat["kind"][:5] != sca["kind"][:5] and not (
            gat["kind"] in ("gather", "block_gather") and sca["kind"] in ("scatter", "block_scatter")
            and gat["kind"].startswith("block") == sca["kind"].startswith("block")):
        return False
    da, db = gat["attrs"].get("dist"), sca["attrs"].get("dist")
    if (da is None) != (db is None):
        return False
    if da is not None and (list(da["grid"]) != list(db["grid"]) or da["scheme"] != db["scheme"]):
        return False
    sa = [str(x) for x in D.cont[x_local]["shape"]]
    sb = [str(x) for x in D.cont[xp_local]["shape"]]
    if len(sa) != len(sb):
        return False
    for p, q in zip(sa, sb):
        if p == q:
            continue
        ip, iq = D.dsym.get(p), D.dsym.get(q)
        if ip is None or iq is None:
            return False
        if (_norm(symexpr.parse(ip["extent"])) != _norm(symexpr.parse(iq["extent"]))
                or ip["dim"] != iq["dim"] or ip["grid"] != iq["grid"]):
            return False
    return True


def _norm(e):
    from .validate import normalize

    return normalize(e)


def _same_subset(a, b) -> bool:
    return len(a) == len(b) and all(
        _norm(x) == _norm(y) for da, db in zip(a, b) for x, y in zip(da, db))


def remove_redundant_comm(doc) -> dict:
    """Remove gather -> T -> scatter pairs with provably equal distributions
     from a schema-v1 document in place — or from a
    reference ``Sdfg`` in place; returns the report (pass name -> count)."""
    if _is_reference_sdfg(doc):
        d = as_doc(doc)
        d.setdefault("dist_symbols", dict(getattr(doc, "_b2_dist_symbols", {}) or {}))
        rep = remove_redundant_comm(d)
        _write_back(doc, d)
        return _Report(rep)
    return _Report(_remove_redundant_comm(doc))


class _Report(dict):
    """A report dict that also reads like the reference's PassReport."""

    @property
    def applications(self):
        return self


def _remove_redundant_comm(doc: dict) -> dict:
    D = _Doc(doc)
    changed = True
    while changed:
        changed = False
        sites = {}  # container -> list of (state, node, role)
        for st in doc["states"]:
            for n in st["nodes"]:
                if n["type"] == "access":
                    sites.setdefault(n["container"], []).append((st, n))
        for st in doc["states"]:
            for gat in st["nodes"]:
                if gat["type"] != "library" or gat["kind"] not in ("gather", "block_gather"):
                    continue
                ge_in = [e for e in st["edges"] if e["dst"] == gat["id"] and "memlet" in e]
                ge_out = [e for e in st["edges"] if e["src"] == gat["id"] and "memlet" in e]
                if len(ge_in) != 1 or len(ge_out) != 1:
                    continue
                x_local, _ = _parse_memlet(ge_in[0]["memlet"])
                T, t_sub = _parse_memlet(ge_out[0]["memlet"])
                tc = D.cont.get(T)
                if tc is None or not tc.get("transient") or tc.get("storage") == "distributed_local":
                    continue
                # T: exactly this writer and one reader, a matching scatter
                readers = []
                for st2, acc in sites.get(T, []):
                    for e in st2["edges"]:
                        if e["src"] == acc["id"] and "memlet" in e:
                            readers.append((st2, e))
                writers = [(st2, e) for st2, acc in sites.get(T, []) for e in st2["edges"]
                           if e["dst"] == acc["id"]]
                if len(writers) != 1 or len(readers) != 1:
                    continue
                st2, re_ = readers[0]
                sca = next(x for x in st2["nodes"] if x["id"] == re_["dst"])
                if sca["type"] != "library" or sca["kind"] not in ("scatter", "block_scatter"):
                    continue
                if not _same_subset(_parse_memlet(re_["memlet"])[1], t_sub):
                    continue
                so = [e for e in st2["edges"] if e["src"] == sca["id"] and "memlet" in e]
                if len(so) != 1:
                    continue
                xp_local, _ = _parse_memlet(so[0]["memlet"])
                if not _same_dist(D, x_local, xp_local, gat, sca):
                    continue
                if not _chain_states(doc, st["label"], st2["label"]):
                    continue
                # X must have a single writer and X' no other writer
                xw = [1 for s_ in doc["states"] for acc in s_["nodes"] if acc["type"] == "access"
                      and acc["container"] == x_local
                      for e in s_["edges"] if e["dst"] == acc["id"]]
                xpw = [1 for s_ in doc["states"] for acc in s_["nodes"] if acc["type"] == "access"
                       and acc["container"] == xp_local
                       for e in s_["edges"] if e["dst"] == acc["id"]]
                if len(xw) != 1 or len(xpw) != 1:
                    continue
                _rewire(D, st, gat, st2, sca, x_local, xp_local, T)
                D.count("remove_redundant_comm")
                changed = True
                break
            if changed:
                break
    return D.report


def _rewire(D, st, gat, st2, sca, x_local, xp_local, T):
    # drop the gather (and T's access nodes), the scatter; X' -> X
    for s_, node in ((st, gat), (st2, sca)):
        s_["edges"] = [e for e in s_["edges"] if e["src"] != node["id"] and e["dst"] != node["id"]]
        s_["nodes"] = [x for x in s_["nodes"] if x["id"] != node["id"]]
    xshape = D.cont[x_local]["shape"]
    xpshape = D.cont[xp_local]["shape"]
    sym_map = {q: p for p, q in zip(xshape, xpshape) if p != q}
    for s_ in D.d["states"]:
        for n in s_["nodes"]:
            if n["type"] == "access" and n["container"] == xp_local:
                n["container"] = x_local
            if n["type"] == "map_entry" and sym_map:
                n["params"] = [[p, _rename(r, sym_map)] for p, r in n["params"]]
        for e in s_["edges"]:
            if "memlet" in e:
                cont, sub = _parse_memlet(e["memlet"])
                if cont == xp_local:
                    cont = x_local
                e["memlet"] = _rename(_memlet(cont, sub) if sub or cont != xp_local else
                                      f"{cont}[]", sym_map) if (cont == x_local or sym_map) else \
                    e["memlet"]
        used = {e["src"] for e in s_["edges"]} | {e["dst"] for e in s_["edges"]}
        s_["nodes"] = [n for n in s_["nodes"] if not (n["type"] == "access" and n["container"] == T
                                                     and n["id"] not in used)]
    D.d["containers"] = [c for c in D.d["containers"] if c["name"] not in (xp_local,)]
    D.cont.pop(xp_local, None)
    still = any(n["type"] == "access" and n["container"] == T
                for s_ in D.d["states"] for n in s_["nodes"])
    if not still:
        D.d["containers"] = [c for c in D.d["containers"] if c["name"] != T]
        D.cont.pop(T, None)


def _rename(text, sym_map):
    if not sym_map:
        return text
    out = text
    for q, p in sym_map.items():
        out = _replace_word(out, q, p)
    return out


def _replace_word(text, old, new):
    import re

    return re.sub(rf"\b{re.escape(old)}\b", new, text)


# ---------------------------------------------------------------------------


def as_doc(g) -> dict:
    """A deep copy of ``g`` as a schema-v1 document."""
    if isinstance(g, dict):
        return copy.deepcopy(g)
    if isinstance(g, sdfg.Graph):
        if g.doc is None:
            raise DistError("graph has no document")
        return copy.deepcopy(g.doc)
    if isinstance(g, str):
        return json.loads(g)
    return copy.deepcopy(sdfg.as_graph(g).doc)


class PassResult(tuple):
    """(document, report) — also the reference's PassReport shape:
    ``.applications`` is the report (pass name -> count), ``.doc`` the
    rewritten schema-v1 document."""

    def __new__(cls, doc, report):
        r = super().__new__(cls, (doc, report))
        r.doc, r.applications = doc, report
        return r


def _canonical_ids(doc: dict) -> dict:
    """Node ids renumbered 0..n-1 per state (the reference serializer indexes
    nodes by position, serialize.py:229)."""
    doc = copy.deepcopy(doc)
    for st in doc["states"]:
        remap = {n["id"]: i for i, n in enumerate(st["nodes"])}
        for n in st["nodes"]:
            n["id"] = remap[n["id"]]
            if n.get("type") == "map_exit":
                n["entry"] = remap[n["entry"]]
        for e in st["edges"]:
            e["src"], e["dst"] = remap[e["src"]], remap[e["dst"]]
    return doc


def _is_reference_sdfg(g) -> bool:
    return (not isinstance(g, (dict, str, sdfg.Graph)) and hasattr(g, "states")
            and type(g).__module__.split(".")[0] == "sdfgkit")


def _write_back(g, doc: dict) -> None:
    """Rewrite a reference ``Sdfg`` in place (the reference passes mutate
    their argument): the document goes through the reference's own
    serializer; the local-extent symbols ride along on the object."""
    ser = importlib.import_module(type(g).__module__.split(".")[0] + ".serialize")
    new = ser.from_dict(_canonical_ids(doc))
    g.__dict__.clear()
    g.__dict__.update(new.__dict__)
    g._b2_dist_symbols = dict(doc.get("dist_symbols") or {})


def distribute(g, grid, blocks=None) -> PassResult:
    """distribute_elementwise + expand_matmul_distributed; returns (new
    document, report).  A reference ``Sdfg`` argument is also rewritten in
    place, like the reference pass."""
    doc = as_doc(g)
    rep = {}
    for k, v in expand_matmul_distributed(doc, grid).items():
        rep[k] = rep.get(k, 0) + v
    for k, v in distribute_elementwise(doc, grid, blocks).items():
        rep[k] = rep.get(k, 0) + v
    if _is_reference_sdfg(g):
        _write_back(g, doc)
    return PassResult(doc, rep)


def distribution_pipeline(g, grid) -> PassResult:
    doc, rep = distribute(as_doc(g), grid)
    for k, v in remove_redundant_comm(doc).items():
        rep[k] = rep.get(k, 0) + v
    if _is_reference_sdfg(g):
        _write_back(g, doc)
    return PassResult(doc, rep)


def local_bindings(doc: dict, grid, bindings: dict, rank: int) -> dict:
    """Per-rank values of the local-extent symbols (block distribution;
    extents the grid does not divide are an error)."""
    _dims(grid)
    out = dict(bindings)
    for name, info in doc.get("dist_symbols", {}).items():
        ext = symexpr.evaluate(symexpr.parse(info["extent"]), bindings)
        gd, d = info["grid"], info["dim"]
        if d is None or d >= len(gd):
            out[name] = ext
            continue
        if ext % gd[d]:
            raise DistError(f"extent {ext} is not covered by grid dimension {gd[d]} "
                            "(divisible block sizes required)")
        out[name] = ext // gd[d]  # block: every rank holds the same extent
    _ = rank
    return out
