"""Device loop regions: host-driven `for ... in range(...)` loops of the state
machine compiled into ONE kernel.

The reference runs every state of a lowered range loop on the host, one
state transition per iteration (Machine.run, pkg/src/sdfgkit/interp.py:
240-263; loops are lowered as guard/body/latch states by frontend/lower.py:
310-348).  For loops whose bodies are only map/tasklet ops that is one kernel
launch per iteration (go_fast: 12000; softmax's row max: N*H*SM*SM).  Here a
maximal such loop nest becomes a single launch:

* the outermost loops whose iterations are provably independent (every
  container written in the body is indexed, in one dimension, by exactly the
  loop variable in every access — the legality the reference's LoopToMap
  should have checked; its own LoopToMap miscompiles softmax)
  are distributed over threads,
* the rest of the nest runs sequentially in each thread as structured C
  (loops, straight-line states, symbol assignments) in program order.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import plan as P, scalar, sdfg, symexpr


@dataclass
class Loop:
    guard: str
    var: str
    step: int
    cond: tuple  # scalar expr entering the body
    body_entry: str
    exit: str
    entry_edge: sdfg.Transition
    back_edge: sdfg.Transition
    body: set = field(default_factory=set)  # chain heads inside (not the guard)
    t_in: sdfg.Transition | None = None  # guard -> body (may init an inner loop var)
    t_out: sdfg.Transition | None = None  # guard -> exit (may step an outer loop var)


@dataclass
class Region:
    loop: Loop
    par: list  # perfectly nested parallel loops, outermost first
    heads: set  # every chain head executed inside the region (guard included)
    idx: int = -1
    spec: object = None
    block: bool = False  # one CTA runs the whole nest, its maps spread over the threads
    private: set = field(default_factory=set)  # transients privatised per parallel iteration


def _trans_in(planner: P.Planner) -> dict:
    ins: dict[str, list] = {}
    for t in planner.g.transitions:
        ins.setdefault(t.dst, []).append(t)
    return ins


def find_loops(planner: P.Planner) -> dict[str, Loop]:
    g = planner.g
    heads = set(planner.ops)
    tail_of = {planner.chain_end[h]: h for h in heads}
    ins = _trans_in(planner)
    loops: dict[str, Loop] = {}
    for h in heads:
        outs = g.out_transitions(planner.chain_end[h])
        if planner.ops[h] or len(outs) != 2:
            continue
        if any(t.condition is None for t in outs):
            continue
        into = ins.get(h, [])
        if len(into) != 2:
            continue
        for t_in, t_out in ((outs[0], outs[1]), (outs[1], outs[0])):
            body = _reach(planner, t_in.dst, h, tail_of)
            if body is None or t_out.dst in body:
                continue
            back = [t for t in into if tail_of.get(t.src) in body or t.src in body]
            entry = [t for t in into if t not in back]
            if len(back) != 1 or len(entry) != 1:
                continue
            ba = back[0].assignments
            if len(ba) != 1:
                continue
            v, e = next(iter(ba.items()))
            a = symexpr.affine(e, (v,), {})
            if a is None or a[1] != {v: 1} or a[0] == 0:
                continue
            if v not in scalar.free_names(t_in.condition) or v not in entry[0].assignments:
                continue
            loops[h] = Loop(h, v, a[0], t_in.condition, t_in.dst, t_out.dst, entry[0], back[0],
                            body, t_in, t_out)
            break
    return loops


def _reach(planner, start, stop, tail_of):
    """Chain heads reachable from ``start`` without passing ``stop``."""
    g = planner.g
    seen = set()
    stack = [start]
    while stack:
        h = stack.pop()
        if h == stop or h in seen:
            continue
        if h not in planner.ops:
            return None
        seen.add(h)
        for t in g.out_transitions(planner.chain_end[h]):
            stack.append(t.dst)
    return seen


def _compilable(planner, loop: Loop, loops: dict, maps: bool = False) -> bool:
    g = planner.g
    for h in loop.body:
        if h in loops:
            inner = loops[h]
            if not inner.body <= loop.body or inner.exit not in loop.body | {loop.guard}:
                return False
            continue
        # inside some inner loop's body: checked through that loop as well.
        # Only scalar (top-level tasklet) ops: loops around real maps stay
        # host-driven, each map a full-width kernel in the captured graph —
        # unless every map is small enough for one CTA (``maps``: block
        # regions, below)
        for op in planner.ops[h]:
            if maps == "par" and isinstance(op, P.LibOp) and _reduce_lib_ok(op):
                continue
            if not isinstance(op, P.MapGroup):
                return False
            if op.schedule != "scalar" and not (maps and _block_map_ok(planner, op)):
                return False
        outs = g.out_transitions(planner.chain_end[h])
        if len(outs) != 1 or outs[0].condition is not None:
            return False
        if outs[0].dst not in loop.body | {loop.guard}:
            return False
    for t in g.transitions:
        if t.condition is not None and any(n in g.containers for n in scalar.free_names(t.condition)):
            if t.src in {planner.chain_end[h] for h in loop.body | {loop.guard}}:
                return False
    return True


def _accesses(planner, heads) -> list:
    out = []
    for h in heads:
        for op in planner.ops[h]:
            for m in op.members:
                for acc in planner.member_accesses(m, op.params):
                    out.append((op, m, acc))
    return out


def _independent(planner, loop: Loop, par_vars: list) -> bool:
    """Each container written in the body is, in some dimension, indexed by
    exactly ``loop.var`` (same affine form in every access of the body)."""
    keys_extra = tuple(par_vars)
    writes: dict[str, list] = {}
    allacc: dict[str, list] = {}
    for h in loop.body | {loop.guard}:
        for op in planner.ops[h]:
            if isinstance(op, P.LibOp):
                st, n = op.state, op.node
                accs = [[(e.memlet.container, e.dst is not n, e.memlet.wcr, e.memlet.subset)
                         for e in st.in_edges(n) + st.out_edges(n) if e.memlet is not None]]
            else:
                accs = [_raw_accesses(planner, m) for m in op.members]
            for acc in accs:
                for (c, w, wcr, subset) in acc:
                    allacc.setdefault(c, []).append((w, wcr, subset))
                    if w:
                        writes.setdefault(c, []).append(wcr)
    for c, wl in writes.items():
        if planner.placement.get(c) == "reg":
            continue  # op-local register: private per thread
        if any(w is not None for w in wl):
            return False
        accs = allacc[c]
        ok_dim = False
        ndim = len(accs[0][2])
        for d in range(ndim):
            forms = set()
            good = True
            for (_, _, subset) in accs:
                b, e, _ = subset[d]
                fb = symexpr.affine(b, (loop.var,) + keys_extra, planner.fixed)
                fe = symexpr.affine(e, (loop.var,) + keys_extra, planner.fixed)
                if fb is None or fb != fe or fb[1].get(loop.var) != 1:
                    good = False
                    break
                forms.add((fb[0], tuple(sorted(fb[1].items()))))
            if good and len(forms) == 1:
                ok_dim = True
                break
        if not ok_dim:
            return False
    return True


def _raw_accesses(planner, m: P.Member):
    """(container, is_write, wcr, subset) for every memlet of a member."""
    st = m.state
    out = []

    def tasklet(t):
        for e in st.in_edges(t):
            if e.memlet is not None:
                out.append((e.memlet.container, False, None, e.memlet.subset))
        for e in st.out_edges(t):
            if e.memlet is not None:
                out.append((e.memlet.container, True, e.memlet.wcr, e.memlet.subset))

    def scope(entry):
        for c in P._scope_children(st, entry):
            if isinstance(c, sdfg.Tasklet):
                tasklet(c)
            elif isinstance(c, sdfg.MapEntry):
                scope(c)
            elif isinstance(c, sdfg.Library):
                for e in st.in_edges(c) + st.out_edges(c):
                    if e.memlet is not None:
                        out.append((e.memlet.container, e.dst is not c, e.memlet.wcr,
                                    e.memlet.subset))

    if m.tasklet is not None:
        tasklet(m.tasklet)
    else:
        scope(m.entry)
    return out


def _perfect_child(planner, loop: Loop, loops: dict) -> Loop | None:
    """The loop directly nested in ``loop`` when the body is nothing else."""
    g = planner.g
    h = loop.body_entry
    seen = set()
    walked = []
    while h not in loops:
        if h in seen or planner.ops.get(h):
            return None
        seen.add(h)
        outs = g.out_transitions(planner.chain_end[h])
        if len(outs) != 1 or outs[0].condition is not None:
            return None
        walked.append(outs[0])
        h = outs[0].dst
    inner = loops[h]
    if any(set(t.assignments) - {inner.var} for t in walked + [loop.t_in]):
        return None
    if set(inner.t_out.assignments) - {loop.var}:
        return None
    # after the inner loop exits we must go straight back to our guard
    x = inner.exit
    while x != loop.guard:
        if planner.ops.get(x) or x in seen:
            return None
        seen.add(x)
        outs = g.out_transitions(planner.chain_end[x])
        if len(outs) != 1 or outs[0].condition is not None:
            return None
        if outs[0] is not loop.back_edge and outs[0].assignments:
            return None
        x = outs[0].dst
    return inner


def _block_map_ok(planner, op) -> bool:
    """A parallel map one CTA can sweep per loop iteration: constant ranges
    of at most BLOCK_MAX_POINTS points, no WCR writes (threads would race on
    the targets) and no library nodes in its scope."""
    from . import codegen

    if op.schedule != "parallel":
        return False
    npts = 1
    for r in op.ranges:
        cr = codegen._const_range(planner, r)
        if cr is None:
            return False
        npts *= cr[2]
    if npts > BLOCK_MAX_POINTS:
        return False
    for m in op.members:
        acc = _raw_accesses(planner, m)
        if any(w and wcr is not None for (_, w, wcr, _) in acc):
            return False
        if any(planner.placement.get(c) == "private" for (c, _, _, _) in acc):
            return False
        if m.entry is not None and any(isinstance(n, sdfg.Library)
                                       for n in P._scope_children(m.state, m.entry)):
            return False
    return True


def _reduce_lib_ok(op) -> bool:
    """A whole-array REDUCE library node (doitgen's sum over a transient row):
    one sequential in-thread loop inside a region (codegen.library_in_scope)."""
    n = op.node
    return (n is not None and n.kind == "reduce" and n.attrs.get("axes") is None
            and not op.fused and op.prologue is None and op.rowpass is None)


def _has_parallel_map(planner, loop: Loop) -> bool:
    return any(isinstance(op, P.MapGroup) and op.schedule == "parallel"
               for h in loop.body for op in planner.ops[h])


def _nested_map_loop(planner, loop: Loop, loops: dict) -> bool:
    """An inner loop of ``loop`` iterates maps: the launch count is the
    product of trip counts (adi: TSTEPS x 4 x (N - 2)).  A single loop
    around maps (a stencil's time loop) keeps one full-width kernel per map
    in the captured graph."""
    return any(h in loops and h != loop.guard and _has_parallel_map(planner, loops[h])
               for h in loop.body)


def find_regions(planner: P.Planner) -> list[Region]:
    if not LOOP_REGIONS:
        return []
    loops = find_loops(planner)
    comp = {h: l for h, l in loops.items() if _compilable(planner, l, loops)}
    roots = [l for h, l in comp.items()
             if not any(h in other.body for oh, other in comp.items() if oh != h)]
    regions = []
    for root in roots:
        par = []
        cur = root
        while cur is not None and _independent(planner, cur, [l.var for l in par]):
            par.append(cur)
            cur = _perfect_child(planner, cur, loops)
            if cur is not None and cur.guard not in comp:
                cur = None
        reg = Region(root, par, root.body | {root.guard})
        if _symbols_escape(planner, reg):
            continue
        regions.append(reg)
    if BLOCK_REGIONS:
        regions += _block_regions(planner, loops, regions)
    if MAP_REGIONS:
        regions += _map_regions(planner, loops, regions)
    return regions


def _op_containers(planner, op) -> set:
    if isinstance(op, P.MapGroup):
        names = set()
        for m in op.members:
            names |= {c for (c, _, _, _) in _raw_accesses(planner, m)}
        return names
    if isinstance(op, P.LibOp) and op.node is not None:
        return {e.memlet.container for e in op.state.in_edges(op.node) + op.state.out_edges(op.node)
                if e.memlet is not None}
    return set(planner.g.containers)  # copies / nested graphs: treat as touching everything


def _privatisable(planner, root: Loop, loops: dict) -> set:
    """Transients only the body of ``root`` touches whose first access in
    each iteration is a map writing the whole container point by point
    (doitgen's tmp0[k] = A[r, q, k] * C4[k, p], k over all of tmp0): a
    per-iteration private copy is then exact."""
    from . import codegen

    heads = root.body | {root.guard}
    touched: dict = {}
    for h, ops in planner.ops.items():
        for op in ops:
            for c in _op_containers(planner, op):
                touched.setdefault(c, set()).add(h)
    out = set()
    for c, hs in touched.items():
        cont = planner.g.containers.get(c)
        if cont is None or not cont.transient or not hs <= heads or c in planner.host_read:
            continue
        if planner.placement.get(c) != "memory":
            continue
        shape = [symexpr.evaluate(d, planner.fixed) for d in cont.shape] if cont.shape else []
        if not shape or any(not isinstance(x, int) for x in shape) or \
                __import__("math").prod(shape) > PRIVATE_MAX_ELEMS:
            continue
        # the first op of the body (program order) touching c writes all of it
        first = None
        cur, seen = root.body_entry, set()
        while cur in root.body and cur not in seen and first is None:
            seen.add(cur)
            for op in planner.ops[cur]:
                if c in _op_containers(planner, op):
                    first = op
                    break
            if cur in loops:  # into the nested loop's body
                cur = loops[cur].body_entry
                continue
            outs = planner.g.out_transitions(planner.chain_end[cur])
            cur = outs[0].dst if len(outs) == 1 else None
        if not isinstance(first, P.MapGroup) or first.schedule != "parallel" \
                or len(first.members) != 1:
            continue
        m = first.members[0]
        acc = [a for a in _raw_accesses(planner, m) if a[0] == c]
        if not acc or not acc[0][1] or acc[0][2] is not None:
            continue
        ranges = [codegen._const_range(planner, r) for r in first.ranges]
        sub = acc[0][3]
        full = len(sub) == len(shape)
        for d, (b, e, _) in enumerate(sub if full else []):
            names = symexpr.free_symbols(b)
            if b != e or len(names) != 1:
                full = False
                break
            q = next(iter(names))
            gp = m.rename.get(q, q)
            if gp not in first.params or b != ("s", q):
                full = False
                break
            r = ranges[first.params.index(gp)]
            if r is None or r != (0, 1, shape[d]):
                full = False
                break
        if full:
            out.add(c)
    return out


def _map_regions(planner, loops: dict, regions: list) -> list:
    """Perfectly nested independent loops around small maps and whole-array
    REDUCEs (doitgen.raw: r, q, p around a 256-point map into tmp0 and a
    sum of tmp0): the reference runs NR x NQ x NP host iterations, a
    launch-per-map backend two kernels per iteration.  Here one thread per
    (r, q, p) runs the body sequentially with its own copy of each
    privatisable transient.  Only when the parallel trip count fills the GPU
    and the body has no sequential loops (counters: one body walk times the
    trip count)."""
    taken = set()
    for r in regions:
        taken |= r.heads
    out = []
    for h, root in loops.items():
        if (root.body | {h}) & taken or any(h in o.body for oh, o in loops.items() if oh != h):
            continue
        if not _compilable(planner, root, loops, maps="par"):
            continue
        priv = _privatisable(planner, root, loops)
        saved = {c: planner.placement[c] for c in priv}
        for c in priv:
            planner.placement[c] = "reg"  # private per thread: no cross-iteration effect
        try:
            par, cur = [], root
            while cur is not None and _independent(planner, cur, [l.var for l in par]):
                par.append(cur)
                cur = _perfect_child(planner, cur, loops)
        finally:
            planner.placement.update(saved)
        if not par:
            continue
        inner = par[-1]
        if any(x in loops for x in inner.body):
            continue  # sequential loops inside the body
        env = dict(planner.fixed)
        n = 1
        try:
            for L in par:
                v0 = symexpr.evaluate(L.entry_edge.assignments[L.var], env)
                vals = trip(L, v0, env)
                env[L.var] = vals[0] if vals else v0
                n *= len(vals)
        except Exception:
            continue
        if n < MAP_REGION_MIN_PAR:
            continue
        reg = Region(root, par, root.body | {root.guard}, private=priv)
        if _symbols_escape(planner, reg):
            continue
        out.append(reg)
    return out


def _block_regions(planner, loops: dict, regions: list) -> list:
    """Host loops whose bodies hold small maps (adi's column / row sweeps:
    one 398-point map per step of a 398-step j loop): the reference runs one
    state transition per iteration (interp.py:240-263), a launch-per-map
    backend one kernel per iteration.  Here the outermost such loop nest is
    ONE single-CTA kernel: control flow and symbols uniform across the CTA,
    every map's points spread over the threads, a barrier after every op
    (program order, so results are bitwise those of the launch sequence)."""
    taken = set()
    for r in regions:
        taken |= r.heads
    cand = {h: l for h, l in loops.items()
            if not (l.body | {h}) & taken and _compilable(planner, l, loops, maps=True)
            and _nested_map_loop(planner, l, loops)}
    out = []
    for h, root in cand.items():
        if any(h in other.body for oh, other in cand.items() if oh != h):
            continue
        reg = Region(root, [], root.body | {root.guard}, block=True)
        if _symbols_escape(planner, reg):
            continue
        out.append(reg)
    return out


def region_transitions(planner, reg: Region) -> list:
    tails = {planner.chain_end[h] for h in reg.heads}
    return [t for t in planner.g.transitions if t.src in tails]


def assigned_symbols(planner, reg: Region) -> set:
    out = set()
    for t in region_transitions(planner, reg):
        out |= set(t.assignments)
    return out


def _symbols_escape(planner, reg: Region) -> bool:
    """Symbols assigned inside the region (other than the root loop variable,
    whose final value the host recomputes) must not be read outside it."""
    inner = assigned_symbols(planner, reg) - {reg.loop.var}
    if not inner:
        return False
    tails = {planner.chain_end[h] for h in reg.heads}
    for t in planner.g.transitions:
        if t.src in tails:
            continue
        used = set()
        for v in t.assignments.values():
            used |= symexpr.free_symbols(v)
        if t.condition is not None:
            used |= scalar.free_names(t.condition)
        if used & inner:
            return True
    for h, ops in planner.ops.items():
        if h in reg.heads:
            continue
        for op in ops:
            if isinstance(op, P.MapGroup):
                for m in op.members:
                    shadow = set()
                    if m.entry is not None:
                        shadow |= set(m.entry.param_names)
                        for n in m.state.nodes:
                            if isinstance(n, sdfg.MapEntry):
                                shadow |= set(n.param_names)
                    for (c, w, wcr, subset) in _raw_accesses(planner, m):
                        for d in subset:
                            for x in d:
                                if (symexpr.free_symbols(x) - shadow) & inner:
                                    return True
    return False


LOOP_REGIONS = True
BLOCK_REGIONS = True
BLOCK_MAX_POINTS = 4096  # points of one map inside a block region (one CTA sweeps them)
MAP_REGIONS = True
MAP_REGION_MIN_PAR = 148 * 64  # parallel iterations a thread-per-iteration region needs
PRIVATE_MAX_ELEMS = 4096  # elements of a per-thread private transient (local memory)


def trip(loop: Loop, init: int, env: dict) -> list[int]:
    """Values the loop variable takes (condition must be v <op> E)."""
    c = loop.cond
    if c[0] != "bin" or c[2] != ("ref", loop.var):
        raise P.PlanError("loop condition is not of the form var <op> bound")
    bound = scalar.evaluate(c[3], env)
    op = c[1]
    step = loop.step
    if op == "<":
        return list(range(init, bound, step)) if step > 0 else []
    if op == "<=":
        return list(range(init, bound + 1, step)) if step > 0 else []
    if op == ">":
        return list(range(init, bound, step)) if step < 0 else []
    if op == ">=":
        return list(range(init, bound - 1, step)) if step < 0 else []
    if op == "!=":
        return list(range(init, bound, step))
    raise P.PlanError(f"unsupported loop condition operator {op}")
