"""Planner: lowers a program graph into a per-state list of device ops.

The reference executes every map scope point by point in lexicographic order
(``Machine.exec_map``, pkg/src/sdfgkit/interp.py:420-441).  On B200 each
top-level scope becomes ONE kernel launch of a hand-written family template
whose body is the scope's tasklet chain compiled by NVRTC:

* ``MapGroup``  — parallel map (or run of fused maps / top-level tasklets)
  -> generic map family (codegen.py); chains of elementwise maps over the same
  iteration space that communicate through transients are fused here (the
  backend-side fusion SURVEY.md §7.4 calls for: the reference's own
  ``subgraph_fusion`` crashes on heat_3d, §0).
* ``CopyOp``    — access->access copy (interp.py:383-398) -> b2_copy_view
* ``MatmulOp``  — MATMUL (interp.py:450-460) -> rowpass family (2D@1D, 1D@2D
  and the fused gemver/atax/bicg passes) or b2_gemm_f64/f32 (2D@2D)
* ``ReduceOp``  — REDUCE (interp.py:461-473) -> b2_reduce
* ``TransposeOp`` — TRANSPOSE (interp.py:474-480) -> b2_copy_view
* ``NestedOp``  — nested graph (interp.py:491-517) -> recursive executor

Transient placement (replaces ``Machine.prepare`` allocation, interp.py:
199-221 and ``transient_mitigation``, autoopt.py:609-635): a transient whose
every access lies in one fused kernel at one point per map point becomes a
register; one accessed only inside one parallel kernel is privatised per
thread (e.g. doitgen's ``tmp0`` written by an inner map); everything else is
an HBM buffer that lives for the whole run.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import scalar, sdfg, symexpr


class PlanError(NotImplementedError):
    """A graph construct the B200 backend does not implement (raised at plan
    time; there is no CPU fallback)."""


# ---------------------------------------------------------------------------
# canonical affine forms (for range equality and point-access identity)


def canon(e, params: tuple, fixed: dict):
    """Canonical key of an int expression: affine form over ``params`` (map
    params and loop-assigned symbols) after substituting fixed bindings;
    None when not affine."""
    a = symexpr.affine(e, params, fixed)
    if a is None:
        return None
    c0, co = a
    return (c0, tuple(sorted(co.items())))


@dataclass
class Site:
    """One memlet access to a container inside a planned op."""
    op: int
    container: str
    is_write: bool
    wcr: str | None
    depth: int  # 0 = directly in the top-level map scope
    point: tuple | None  # canonical per-dim keys when a single point at depth 0


@dataclass
class Member:
    """One original top-level scope inside a (possibly fused) map group."""
    state: sdfg.State
    entry: sdfg.MapEntry | None  # None for a top-level tasklet
    tasklet: sdfg.Tasklet | None
    rename: dict  # member param name -> group param name


@dataclass
class Op:
    kind: str
    state: sdfg.State
    idx: int = -1


@dataclass
class MapGroup(Op):
    params: list = field(default_factory=list)  # group param names
    ranges: list = field(default_factory=list)  # [(b, e, s)] symexpr (group names)
    schedule: str = "parallel"
    members: list = field(default_factory=list)
    sites: list = field(default_factory=list)
    kernel: object = None  # codegen.KernelSpec after codegen


@dataclass
class CopyOp(Op):
    edge: sdfg.Edge = None


@dataclass
class LibOp(Op):
    node: sdfg.Library = None
    fused: list = field(default_factory=list)  # extra nodes folded into this op
    prologue: MapGroup | None = None
    rowpass: object = None


@dataclass
class NestedOp(Op):
    node: sdfg.Nested = None


def _scope_children(st: sdfg.State, entry: sdfg.MapEntry) -> list:
    parents = st.scope_parents()
    ex = st.exit_of(entry)
    return [n for n in st.topological() if parents.get(n.id) is entry and n is not ex]


class Planner:
    def __init__(self, g: sdfg.Graph, fixed: dict):
        self.g = g
        self.fixed = {k: int(v) for k, v in fixed.items()}
        self.loopish = set()
        for t in g.transitions:
            self.loopish |= set(t.assignments)
        for k in list(self.fixed):
            if k in self.loopish:
                # assigned by a transition: varies during the run
                del self.fixed[k]
        self.ops: dict[str, list[Op]] = {}
        self.all_ops: list[Op] = []
        self.placement: dict[str, str] = {}  # container -> reg | private | memory

    # -- building --------------------------------------------------------------

    def _chains(self) -> dict[str, list[sdfg.State]]:
        """Straight-line runs of states (single unconditional, assignment-free
        transition into a state with one predecessor) are planned as one op
        sequence, so fusion crosses the statement-per-state boundaries of
        un-coarsened graphs (the effect of passes.coarsen, passes.py:759)."""
        indeg: dict[str, int] = {s.label: 0 for s in self.g.states}
        for t in self.g.transitions:
            indeg[t.dst] = indeg.get(t.dst, 0) + 1
        nxt: dict[str, str] = {}
        for st in self.g.states:
            trs = self.g.out_transitions(st.label)
            if (len(trs) == 1 and trs[0].condition is None and not trs[0].assignments
                    and indeg.get(trs[0].dst, 0) == 1 and trs[0].dst != self.g.start
                    and trs[0].dst != st.label):
                nxt[st.label] = trs[0].dst
        inner = set(nxt.values())
        chains = {}
        for st in self.g.states:
            if st.label in inner:
                continue
            chain = [st]
            seen = {st.label}
            cur = st.label
            while cur in nxt and nxt[cur] not in seen:
                cur = nxt[cur]
                seen.add(cur)
                chain.append(self.g.state(cur))
            chains[st.label] = chain
        return chains

    def build(self):
        self.chain_end: dict[str, str] = {}
        for head, chain in self._chains().items():
            ops = []
            for st in chain:
                ops += self._state_ops(st)
            ops = self._fuse(ops)
            ops = self._fuse_blas2(ops)
            for op in ops:
                op.idx = len(self.all_ops)
                self.all_ops.append(op)
            self.ops[head] = ops
            self.chain_end[head] = chain[-1].label
        self._collect_sites()
        self._place()
        from . import loops

        self.regions = loops.find_regions(self)
        self.region_at = {}
        self.in_region: set[int] = set()
        for i, reg in enumerate(self.regions):
            reg.idx = 100000 + i
            self.region_at[reg.loop.guard] = reg
            for h in reg.heads:
                for op in self.ops[h]:
                    self.in_region.add(op.idx)
        return self

    def _state_ops(self, st: sdfg.State) -> list[Op]:
        parents = st.scope_parents()
        ops: list[Op] = []
        for n in st.topological():
            if parents.get(n.id) is not None:
                continue
            if isinstance(n, sdfg.Access):
                for e in st.in_edges(n):
                    if isinstance(e.src, sdfg.Access) and e.memlet is not None:
                        ops.append(CopyOp("copy", st, edge=e))
            elif isinstance(n, sdfg.Tasklet):
                ops.append(MapGroup("map", st, params=[], ranges=[], schedule="scalar",
                                    members=[Member(st, None, n, {})]))
            elif isinstance(n, sdfg.MapEntry):
                sched = "parallel" if n.schedule in ("parallel", "distributed_hint") else "sequential"
                ops.append(MapGroup("map", st, params=list(n.param_names),
                                    ranges=[r for _, r in n.params], schedule=sched,
                                    members=[Member(st, n, None, {p: p for p in n.param_names})]))
            elif isinstance(n, sdfg.MapExit):
                pass
            elif isinstance(n, sdfg.Library):
                if n.kind in sdfg.COMM_KINDS or n.attrs.get("comm"):
                    ops.append(LibOp("comm", st, node=n))
                elif n.kind in ("matmul", "reduce", "transpose"):
                    ops.append(LibOp(n.kind, st, node=n))
                else:
                    raise PlanError(f"unknown library node kind {n.kind}")
            elif isinstance(n, sdfg.Nested):
                ops.append(NestedOp("nested", st, node=n))
            else:
                raise PlanError(f"cannot execute node {type(n).__name__}")
        return ops

    # -- access analysis -------------------------------------------------------

    def member_accesses(self, m: Member, group_params: list) -> list:
        """[(container, is_write, wcr, depth, point_key|None)] in execution order."""
        out = []
        keys = tuple(group_params) + tuple(sorted(self.loopish))

        def point_key(memlet, rename, depth):
            if depth > 0:
                return None
            pk = []
            for b, e, s in memlet.subset:
                kb = canon(_rn(b, rename), keys, self.fixed)
                ke = canon(_rn(e, rename), keys, self.fixed)
                if kb is None or kb != ke:
                    return None
                pk.append(kb)
            return tuple(pk)

        def walk_tasklet(st, t, rename, depth):
            for e in st.in_edges(t):
                if e.memlet is not None:
                    out.append((e.memlet.container, False, None, depth,
                                point_key(e.memlet, rename, depth)))
            for e in st.out_edges(t):
                if e.memlet is not None:
                    out.append((e.memlet.container, True, e.memlet.wcr, depth,
                                point_key(e.memlet, rename, depth)))

        def walk_scope(st, entry, rename, depth):
            for c in _scope_children(st, entry):
                if isinstance(c, sdfg.Tasklet):
                    walk_tasklet(st, c, rename, depth)
                elif isinstance(c, sdfg.MapEntry):
                    inner = dict(rename)
                    for p in c.param_names:
                        inner[p] = p  # shadowing: inner params are not group params
                    walk_scope(st, c, inner, depth + 1)
                elif isinstance(c, sdfg.Library):
                    for e in st.in_edges(c):
                        if e.memlet is not None:
                            out.append((e.memlet.container, False, None, depth + 1, None))
                    for e in st.out_edges(c):
                        if e.memlet is not None:
                            out.append((e.memlet.container, True, e.memlet.wcr, depth + 1, None))
                elif isinstance(c, sdfg.Access):
                    for e in st.in_edges(c):
                        if isinstance(e.src, sdfg.Access) and e.memlet is not None:
                            raise PlanError("access-to-access copy inside a map scope")
                elif isinstance(c, sdfg.Nested):
                    raise PlanError("nested graph inside a map scope")

        if m.tasklet is not None:
            walk_tasklet(m.state, m.tasklet, m.rename, 0)
        else:
            walk_scope(m.state, m.entry, m.rename, 0)
        return out

    # -- fusion of consecutive map groups -----------------------------------------

    def _ranges_equal(self, g: MapGroup, m: MapGroup) -> bool:
        if len(g.params) != len(m.params):
            return False
        keys = tuple(sorted(self.loopish))
        for (b1, e1, s1), (b2, e2, s2) in zip(g.ranges, m.ranges):
            for x, y in ((b1, b2), (e1, e2), (s1, s2)):
                cx, cy = canon(x, keys, self.fixed), canon(y, keys, self.fixed)
                if cx is None or cx != cy:
                    return False
        return True

    def _fusible(self, g: MapGroup, m: MapGroup) -> dict | None:
        if g.schedule == "scalar" and m.schedule == "scalar":
            return {}
        if g.schedule != "parallel" or m.schedule != "parallel":
            return None
        if not self._ranges_equal(g, m):
            return None
        rename = dict(zip(m.params, g.params))
        mm = m.members[0]
        m_acc = self.member_accesses(Member(mm.state, mm.entry, mm.tasklet, rename), g.params)
        g_acc = []
        for gm in g.members:
            g_acc += self.member_accesses(gm, g.params)
        g_by: dict[str, list] = {}
        for a in g_acc:
            g_by.setdefault(a[0], []).append(a)
        m_by: dict[str, list] = {}
        for a in m_acc:
            m_by.setdefault(a[0], []).append(a)
        for c in set(g_by) & set(m_by):
            acc = g_by[c] + m_by[c]
            if not any(a[1] for a in acc):
                continue  # read by both: fine
            pts = {a[4] for a in acc}
            if None in pts or len(pts) != 1:
                return None
            if any(a[2] is not None for a in acc):
                return None
        return rename

    def _fuse(self, ops: list[Op]) -> list[Op]:
        out: list[Op] = []
        for op in ops:
            prev = out[-1] if out else None
            if isinstance(op, MapGroup) and isinstance(prev, MapGroup) and len(op.members) == 1:
                rename = self._fusible(prev, op)
                if rename is not None:
                    m = op.members[0]
                    prev.members.append(Member(m.state, m.entry, m.tasklet,
                                               rename if m.entry is not None else {}))
                    continue
            out.append(op)
        return self._rebalance(out)

    def _single(self, g: MapGroup, m: Member) -> MapGroup:
        """A one-member group for ``m`` (a member of ``g``) in m's own names."""
        inv = {gp: mp for mp, gp in m.rename.items()}
        params = [inv.get(p, p) for p in g.params]
        ranges = [tuple(_rn(x, inv) for x in r) for r in g.ranges]
        return MapGroup("map", m.state, params=params, ranges=ranges, schedule=g.schedule,
                        members=[Member(m.state, m.entry, m.tasklet,
                                        {p: p for p in params} if m.entry is not None else {})])

    def _rebalance(self, ops: list[Op]) -> list[Op]:
        """Greedy fusion can swallow the first map of the NEXT sweep (e.g.
        heat_3d's ``tmp = 2*B[p]`` right after the sweep that writes B[p]),
        turning its output into an HBM round trip.  Move such trailing
        members to the following group when they fuse there."""
        changed = True
        while changed:
            changed = False
            for i in range(len(ops) - 1):
                g, h = ops[i], ops[i + 1]
                if not (isinstance(g, MapGroup) and isinstance(h, MapGroup)):
                    continue
                if len(g.members) < 2 or g.schedule != "parallel":
                    continue
                last = g.members[-1]
                writes = {a[0] for a in self.member_accesses(last, g.params) if a[1]}
                h_reads = set()
                for hm in h.members:
                    h_reads |= {a[0] for a in self.member_accesses(hm, h.params) if not a[1]}
                if not (writes & h_reads):
                    continue
                trial = self._single(g, last)
                ok = True
                for hm in h.members:
                    one = self._single(h, hm)
                    rename = self._fusible(trial, one)
                    if rename is None:
                        ok = False
                        break
                    trial.members.append(Member(hm.state, hm.entry, hm.tasklet,
                                                {mp: rename[p] for mp, p in
                                                 zip(one.params, one.params)}
                                                if hm.entry is not None else {}))
                if not ok:
                    continue
                g.members.pop()
                ops[i + 1] = trial
                changed = True
        return ops

    def _fuse_blas2(self, ops: list[Op]) -> list[Op]:
        from . import blas2  # local import: pattern rules live with the rowpass family
        return blas2.fuse(self, ops)

    # -- placement -----------------------------------------------------------------

    def _collect_sites(self):
        self.sites: dict[str, list[Site]] = {}

        self.op_reads: dict[int, set] = {op.idx: set() for op in self.all_ops}
        self.op_writes: dict[int, set] = {op.idx: set() for op in self.all_ops}

        def add(op, c, w, wcr, depth, point):
            self.sites.setdefault(c, []).append(Site(op.idx, c, w, wcr, depth, point))
            (self.op_writes if w else self.op_reads)[op.idx].add(c)
            if w and wcr is not None:
                self.op_reads[op.idx].add(c)

        for op in self.all_ops:
            if isinstance(op, MapGroup):
                for m in op.members:
                    for (c, w, wcr, depth, pt) in self.member_accesses(m, op.params):
                        add(op, c, w, wcr, depth, pt)
            elif isinstance(op, CopyOp):
                e = op.edge
                add(op, e.src.container, False, None, 1, None)
                add(op, e.dst.container, True, e.memlet.wcr, 1, None)
            elif isinstance(op, LibOp):
                nodes = [op.node] + list(op.fused)
                for n in nodes:
                    for e in op.state.in_edges(n) + op.state.out_edges(n):
                        if e.memlet is not None:
                            add(op, e.memlet.container, e.dst is not n, e.memlet.wcr, 1, None)
                if op.prologue is not None:
                    for m in op.prologue.members:
                        for (c, w, wcr, depth, pt) in self.member_accesses(m, op.prologue.params):
                            add(op, c, w, wcr, 1, None)
            elif isinstance(op, NestedOp):
                for e in op.state.in_edges(op.node) + op.state.out_edges(op.node):
                    if e.memlet is not None:
                        add(op, e.memlet.container, e.dst is not op.node, e.memlet.wcr, 1, None)
        # transition conditions may read scalar containers on the host
        self.host_read = set()
        for t in self.g.transitions:
            if t.condition is not None:
                self.host_read |= {n for n in scalar.free_names(t.condition)
                                   if n in self.g.containers}

    def _place(self):
        for name, c in self.g.containers.items():
            sites = self.sites.get(name, [])
            place = "memory"
            if c.transient and sites and name not in self.host_read and c.kind != "stream":
                ops = {s.op for s in sites}
                if len(ops) == 1:
                    op = self.all_ops[next(iter(ops))]
                    if isinstance(op, MapGroup):
                        pts = {s.point for s in sites}
                        first = sites[0]
                        if (None not in pts and len(pts) == 1 and first.is_write
                                and first.wcr is None and first.depth == 0):
                            place = "reg"
                        elif op.schedule == "parallel" and op.params:
                            place = "private"
                        elif op.schedule in ("scalar", "sequential"):
                            place = "memory"
            self.placement[name] = place

    # -- convenience -------------------------------------------------------------

    def shapes(self, bindings: dict | None = None) -> dict:
        env = dict(bindings or self.fixed)
        return {n: tuple(symexpr.evaluate(d, env) for d in c.shape)
                for n, c in self.g.containers.items()}

    def symbol_env(self, env: dict) -> dict:
        e = dict(self.fixed)
        e.update(env)
        return e


def _rn(e, rename: dict):
    """Rename symbols of an expression tree (member params -> group params)."""
    if not rename:
        return e
    k = e[0]
    if k == "c":
        return e
    if k == "s":
        return ("s", rename.get(e[1], e[1]))
    return (k, _rn(e[1], rename), _rn(e[2], rename))


def rn(e, rename):
    return _rn(e, rename)
