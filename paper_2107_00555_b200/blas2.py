"""BLAS-2 planning: MATMUL library nodes in matrix-vector form, and the
gemver / atax / bicg fusions, lowered onto the rowpass family
(csrc/families/rowpass.cuh).

Reference semantics: MATMUL executes ``np.matmul`` on the (squeezed) memlet
views and writes the reshaped result (pkg/src/sdfgkit/interp.py:450-460);
the programs come from the reference corpus (pkg/tests/corpus/gemver.dpy,
atax.dpy, bicg.dpy) lowered by frontend/lower.py:255-266.

Fusion rules over a straight-line op sequence (plan.Planner):
  P1 gemver head  elementwise map writing X[i, j] (full matrix, identity
                  point) immediately followed by ``y @ X`` or ``X @ v``:
                  the map becomes the rowpass prologue (X' written back in
                  the same pass that feeds the product)
  P2 atax         ``t = X @ v`` followed by ``y = t @ X``: one pass, the row
                  dot feeds the column accumulation (coef = dot)
  P3 bicg         ``s = r @ X`` and ``q = X @ p`` adjacent, independent
  P0 single       any lone 2D@1D / 1D@2D product
Operand R of the family must be row-contiguous: a view with unit column
stride is used as is; one with unit row stride is used transposed (the dot
and axpy roles swap).  Anything else stays on b2_gemm_f64.
"""

from __future__ import annotations

import ctypes
import os
import struct

from . import codegen, plan as P, runtime as rt, sdfg, symexpr

TPB = 512
MAX_CW = 8192
TMA_ROWS = os.environ.get("B2_RP_TMA", "1") == "1"  # bulk-copy row ring (rowpass.cuh)
# compensated (Dot2 / double-double) sums in the row pass (rowpass.cuh
# RP_COMP): ~17x closer to the exact result (atax 8000^2: 3.6e-14 vs 6.3e-13
# rel_err against an 80-bit evaluation; the reference's BLAS: 3.5e-12) but
# FP64-issue bound (atax 0.171 vs 0.092 ms), so opt-in
RP_COMP = os.environ.get("B2_RP_COMP", "0") == "1"
# dot-only passes walk the rows bottom-up: a pass that follows another over
# the same matrix (gemver's w = A x after the A update) starts on the rows the
# previous pass left in L2.  Row dots are independent of the row order, so the
# results are bitwise the same; passes with column partials (AXPY) keep the
# forward order their fold relies on.
RP_REV_DOT = os.environ.get("B2_RP_REV", "1") == "1"
SMEM_BUDGET = 220 * 1024


class _View:
    def __init__(self, container, offset, dims):
        self.container = container
        self.offset = offset
        self.dims = dims  # [(len, stride)]


def _view(planner: P.Planner, m: sdfg.Memlet, kept, shapes) -> _View | None:
    try:
        ranges = symexpr.eval_subset(m.subset, planner.fixed)
    except KeyError:
        return None
    shape = shapes[m.container]
    if len(ranges) != len(shape):
        return None
    for d, r in enumerate(ranges):
        if len(r) and (r.start < 0 or r[-1] >= shape[d]):
            return None
    st = codegen._row_major(shape)
    off = sum(r.start * st[d] for d, r in enumerate(ranges))
    dims = [(len(r), st[d] * r.step) for d, r in enumerate(ranges)]
    if kept is not None:
        if len(kept) != len(dims):
            return None
        dims = [dd for dd, k in zip(dims, kept) if k]
    return _View(m.container, off, dims)


class MV:
    """One MATMUL node in matrix-vector form, normalised to R = row-contiguous
    matrix: kind 'dot' (out[m] = R[m,:] . v) or 'axpy' (out[n] = u . R[:, n])."""

    def __init__(self, op, kind, R, vec, out, out_wcr):
        self.op = op
        self.kind = kind
        self.R = R  # (container, offset, M, N, rs)
        self.vec = vec  # _View 1-D
        self.out = out  # _View 1-D
        self.out_wcr = out_wcr


def _mv(planner: P.Planner, op: P.LibOp, shapes) -> MV | None:
    if not isinstance(op, P.LibOp) or op.kind != "matmul" or op.rowpass is not None:
        return None
    n = op.node
    st = op.state
    ins = {e.dst_conn: e for e in st.in_edges(n) if e.memlet is not None}
    outs = [e for e in st.out_edges(n) if e.memlet is not None]
    if "a" not in ins or "b" not in ins or len(outs) != 1:
        return None
    g = planner.g
    for e in (ins["a"], ins["b"], outs[0]):
        if g.containers[e.memlet.container].dtype != "f64":
            return None
    a = _view(planner, ins["a"].memlet, n.attrs.get("a_kept"), shapes)
    b = _view(planner, ins["b"].memlet, n.attrs.get("b_kept"), shapes)
    o = _view(planner, outs[0].memlet, None, shapes)
    if a is None or b is None or o is None:
        return None
    odims = [d for d in o.dims if d[0] != 1]
    if outs[0].memlet.wcr not in (None, "add"):
        return None
    if len(a.dims) == 2 and len(b.dims) == 1:  # X @ v
        (M, rs), (K, cs) = a.dims
        if b.dims[0][0] != K or len(odims) != 1 or odims[0][0] != M:
            return None
        out = _View(o.container, o.offset, odims)
        if cs == 1:
            return MV(op, "dot", (a.container, a.offset, M, K, rs), b, out, outs[0].memlet.wcr)
        if rs == 1:
            return MV(op, "axpy", (a.container, a.offset, K, M, cs), b, out, outs[0].memlet.wcr)
        return None
    if len(a.dims) == 1 and len(b.dims) == 2:  # u @ X
        (K, rs), (N, cs) = b.dims
        if a.dims[0][0] != K or len(odims) != 1 or odims[0][0] != N:
            return None
        out = _View(o.container, o.offset, odims)
        if cs == 1:
            return MV(op, "axpy", (b.container, b.offset, K, N, rs), a, out, outs[0].memlet.wcr)
        if rs == 1:
            return MV(op, "dot", (b.container, b.offset, N, K, cs), a, out, outs[0].memlet.wcr)
        return None
    return None


def _prologue_ok(planner: P.Planner, grp: P.MapGroup, R, shapes):
    """P1: a parallel 2-param map writing only R's container, at the identity
    point over the full matrix, and reading it only there."""
    if not isinstance(grp, P.MapGroup) or grp.schedule != "parallel" or len(grp.params) != 2:
        return None
    cont, off, M, N, rs = R
    shape = shapes[cont]
    if len(shape) != 2 or off != 0:
        return None
    acc = []
    for mem in grp.members:
        acc += planner.member_accesses(mem, grp.params)
    p0, p1 = grp.params
    ident = ((0, ((p0, 1),)), (0, ((p1, 1),)))
    writes = {a[0] for a in acc if a[1]}
    if writes != {cont}:
        return None
    for a in acc:
        if a[0] == cont and (a[4] != ident or a[2] is not None or a[3] != 0):
            return None
    rng = [codegen._const_range(planner, r) for r in grp.ranges]
    if rng != [(0, 1, shape[0]), (0, 1, shape[1])]:
        return None
    # orientation: R rows are X rows (rs == shape[1]) or X columns (transposed)
    if rs == shape[1] and (M, N) == (shape[0], shape[1]):
        return {"m": p0, "n": p1}
    if rs == shape[0] and (M, N) == (shape[1], shape[0]):
        return {"m": p1, "n": p0}
    return None


def _reads(planner, op) -> set:
    out = set()
    if isinstance(op, P.LibOp):
        for e in op.state.in_edges(op.node):
            if e.memlet is not None:
                out.add(e.memlet.container)
    return out


def fuse(planner: P.Planner, ops: list) -> list:
    shapes = planner.shapes()
    out = []
    i = 0
    while i < len(ops):
        op = ops[i]
        nxt = ops[i + 1] if i + 1 < len(ops) else None
        mv = _mv(planner, op, shapes)
        # P1: prologue map + product on the map's matrix
        if isinstance(op, P.MapGroup) and nxt is not None:
            mv2 = _mv(planner, nxt, shapes)
            if mv2 is not None:
                roles = _prologue_ok(planner, op, mv2.R, shapes)
                if roles is not None and mv2.vec.container != mv2.R[0]:
                    rp = RowPass(planner, [mv2], prologue=op, roles=roles)
                    if rp.ok:
                        nxt.rowpass = rp
                        nxt.prologue = op
                        out.append(nxt)
                        i += 2
                        continue
        if mv is not None and nxt is not None:
            mv2 = _mv(planner, nxt, shapes)
            if mv2 is not None and mv2.R == mv.R:
                # P2 atax: dot then axpy whose coefficient vector is the dot output
                if (mv.kind == "dot" and mv2.kind == "axpy" and mv2.vec.container == mv.out.container
                        and mv2.vec.offset == mv.out.offset and mv2.vec.dims == mv.out.dims
                        and mv.out_wcr is None):
                    rp = RowPass(planner, [mv, mv2], coef_from_dot=True)
                    if rp.ok:
                        op.rowpass = rp
                        op.fused = [nxt.node]
                        out.append(op)
                        i += 2
                        continue
                # P3 bicg: independent dot + axpy on the same matrix
                if {mv.kind, mv2.kind} == {"dot", "axpy"}:
                    outs = {mv.out.container, mv2.out.container}
                    if not (outs & (_reads(planner, op) | _reads(planner, nxt))):
                        rp = RowPass(planner, [mv, mv2])
                        if rp.ok:
                            op.rowpass = rp
                            op.fused = [nxt.node]
                            out.append(op)
                            i += 2
                            continue
        if mv is not None:
            rp = RowPass(planner, [mv])
            if rp.ok:
                op.rowpass = rp
        out.append(op)
        i += 1
    return out


class RowPass:
    """A planned rowpass launch (main kernel + deterministic finalize)."""

    def __init__(self, planner: P.Planner, mvs: list, prologue: P.MapGroup | None = None,
                 roles: dict | None = None, coef_from_dot: bool = False):
        self.planner = planner
        self.mvs = mvs
        self.prologue = prologue
        self.roles = roles or {}
        self.coef_from_dot = coef_from_dot
        self.R = mvs[0].R
        self.dot = next((m for m in mvs if m.kind == "dot"), None)
        self.axpy = next((m for m in mvs if m.kind == "axpy"), None)
        cont, off, M, N, rs = self.R
        self.M, self.N, self.rs = M, N, rs
        # prologue reads of 1-D containers indexed by the column alone (gemver's
        # v1[j], v2[j]) are staged once per CTA in shared memory
        self.staged: list[str] = []
        if prologue is not None:
            ncol = self.roles["n"]
            for mem in prologue.members:
                for (c, w, wcr, depth, pt) in planner.member_accesses(mem, prologue.params):
                    if (not w and c != cont and depth == 0 and pt == ((0, ((ncol, 1),)),)
                            and len(planner.g.containers[c].shape) == 1
                            and planner.g.containers[c].dtype == "f64" and c not in self.staged):
                        self.staged.append(c)
        cap = MAX_CW if not self.staged else 4096
        self.cw = min(N, cap)
        self.ctiles = -(-N // self.cw) if N else 1
        self.ok = M > 0 and N > 0 and not (coef_from_dot and self.ctiles > 1)
        if self.dot is not None and self.dot.vec.dims[0][0] != N:
            self.ok = False
        if self.axpy is not None and self.axpy.vec.dims[0][0] != M and not coef_from_dot:
            self.ok = False

    # -- compile ---------------------------------------------------------------

    def source(self, shapes, name: str) -> str:
        M, N, rs, cw = self.M, self.N, self.rs, self.cw
        tpb = int(os.environ.get("B2_RP_TPB", TPB))
        self.tpb = tpb
        kpt = -(-cw // tpb)
        dot, axpy = self.dot, self.axpy
        # TMA row ring when every row slice is a 16-byte aligned, 16-byte
        # multiple (1-D bulk copies); else the register-prefetch kernel
        nst = len(self.staged)
        red = 128 if RP_COMP else 64
        # compensated dot + axpy: the dot vector moves to shared memory
        self.vsmem = RP_COMP and dot is not None and axpy is not None
        vs = cw if self.vsmem else 0
        ring_s = (SMEM_BUDGET // 8 - nst * cw - red - vs) // cw if cw else 0
        off = self.R[1]
        # (gemver's prologue + write-back pass measured faster with the
        # register-prefetch kernel at 2-3 CTAs/SM: 184 vs 254 us)
        self.tma = (TMA_ROWS and self.prologue is None and rs % 2 == 0 and off % 2 == 0
                    and N % 2 == 0 and cw % 2 == 0 and ring_s >= 2)
        if self.tma:
            self.ring = min(4, ring_s)
            stage_base = 0
            self.smem = (nst * cw + red + vs + self.ring * cw) * 8
            self.G = min(M, 148)
        else:
            self.ring = 0
            stage_base = (cw if axpy else 0) * (2 if RP_COMP else 1) + (cw if dot else 0) + red
            smem_doubles = stage_base + cw * nst
            self.smem = smem_doubles * 8
            est_regs = 4 * kpt + 40  # x / xn double arrays + addressing
            blocks_per_sm = max(1, min(4, (200 * 1024) // max(1, self.smem),
                                       65536 // (tpb * est_regs)))
            self.G = min(M, 148 * blocks_per_sm)
        L = []
        L.append(f"#define RP_NAME b2_rp_{name}")
        L.append(f"#define RP_FIN_NAME b2_rpf_{name}")
        for k, v in (("RP_M", M), ("RP_N", N), ("RP_RS", rs), ("RP_CW", cw), ("RP_TPB", tpb),
                     ("RP_KPT", kpt), ("RP_G", self.G), ("RP_CTILES", self.ctiles),
                     ("RP_DOT", int(dot is not None)), ("RP_AXPY", int(axpy is not None)),
                     ("RP_PROLOGUE", int(self.prologue is not None)),
                     ("RP_WRITEBACK", int(self.prologue is not None)),
                     ("RP_TMA", int(self.tma)), ("RP_S", max(1, self.ring)),
                     ("RP_COMP", int(RP_COMP)),
                     ("RP_REV", int(RP_REV_DOT and axpy is None and self.tma)),
                     ("RP_VSMEM", int(self.tma and self.vsmem)),
                     ("RP_NSTAGED", nst)):
            L.append(f"#define {k} {v}LL" if k in ("RP_M", "RP_N", "RP_RS") else f"#define {k} {v}")
        nbase = 8
        pro_src = ""
        if self.prologue is not None:
            cont = self.R[0]
            env = {self.roles["m"]: "m", self.roles["n"]: "n"}
            colstage = {c: f"{stage_base + i * cw}" for i, c in enumerate(self.staged)}
            spec = codegen.point_function(
                self.planner, self.prologue, shapes, name, env, {cont: "x"}, nbase,
                "double rp_elem(const RpArgs &a, const RpRow &rr, b2_ll m, b2_ll n, double x, "
                "int jl)", f"r_{cont}", colstage=colstage)
            self.pro_args = spec.args
            pro_src = spec.source
        else:
            self.pro_args = []
        nargs = nbase + len(self.pro_args)
        L.append("struct RpArgs { long long w[%d]; };" % nargs)
        L.append("struct RpRow { int unused; };")
        L.append("__device__ __forceinline__ void rp_row_setup(const RpArgs &, b2_ll, RpRow &) {}")
        L.append("extern __shared__ double rp_smem[];")
        L.append(pro_src)
        # stage the column vectors of this CTA's column tile
        stage = ["__device__ __forceinline__ void rp_stage_cols(const RpArgs &a, b2_ll c0, int cw, "
                 "int tid) {"]
        for i, c in enumerate(self.staged):
            ai = nbase + self.pro_args.index(("ptr", c))
            stage.append(f"  for (int j = tid; j < cw; j += RP_TPB) rp_smem[{stage_base + i * cw} + j]"
                         f" = ((const double *)a.w[{ai}])[c0 + j];")
        stage.append("}")
        L.append("\n".join(stage))
        if dot is not None:
            vinc = dot.vec.dims[0][1]
            oinc = dot.out.dims[0][1]
            L.append("__device__ __forceinline__ double rp_dot_vec(const RpArgs &a, b2_ll n) "
                     f"{{ return ((const double *)a.w[3])[n * {vinc}LL]; }}")
            add = "*p + d" if dot.out_wcr == "add" else "d"
            if self.ctiles == 1:
                L.append("__device__ __forceinline__ void rp_store_dot(const RpArgs &a, b2_ll m, "
                         f"double d, int) {{ double *p = (double *)a.w[4] + m * {oinc}LL; *p = {add}; }}")
            else:
                L.append("__device__ __forceinline__ void rp_store_dot(const RpArgs &a, b2_ll m, "
                         f"double d, int t) {{ ((double *)a.w[2])[(b2_ll)t * {M}LL + m] = d; }}")
            L.append("__device__ __forceinline__ void rp_store_dot_final(const RpArgs &a, b2_ll m, "
                     f"double d) {{ double *p = (double *)a.w[4] + m * {oinc}LL; *p = {add}; }}")
        else:
            L.append("__device__ __forceinline__ double rp_dot_vec(const RpArgs &, b2_ll) { return 0.0; }")
            L.append("__device__ __forceinline__ void rp_store_dot(const RpArgs &, b2_ll, double, int) {}")
            L.append("__device__ __forceinline__ void rp_store_dot_final(const RpArgs &, b2_ll, double) {}")
        if axpy is not None:
            ainc = axpy.out.dims[0][1]
            add = "*p + s" if axpy.out_wcr == "add" else "s"
            if self.coef_from_dot:
                L.append("__device__ __forceinline__ double rp_coef(const RpArgs &, b2_ll, double d) "
                         "{ return d; }")
            else:
                uinc = axpy.vec.dims[0][1]
                L.append("__device__ __forceinline__ double rp_coef(const RpArgs &a, b2_ll m, double) "
                         f"{{ return ((const double *)a.w[5])[m * {uinc}LL]; }}")
            L.append("__device__ __forceinline__ void rp_store_axpy(const RpArgs &a, b2_ll n, double s) "
                     f"{{ double *p = (double *)a.w[6] + n * {ainc}LL; *p = {add}; }}")
        else:
            L.append("__device__ __forceinline__ double rp_coef(const RpArgs &, b2_ll, double d) "
                     "{ return d; }")
            L.append("__device__ __forceinline__ void rp_store_axpy(const RpArgs &, b2_ll, double) {}")
        return (rt.family_source("prelude.cuh") + "\n" + "\n".join(L) + "\n"
                + rt.family_source("rowpass.cuh"))

    def compile(self, ex):
        name = f"{ex.g.name}_{self.mvs[0].op.idx}"
        src = self.source(ex.buf.shape, name)
        self.kmain = rt.get_kernel(src, f"b2_rp_{name}", max_smem=self.smem)
        self.kfin = rt.get_kernel(src, f"b2_rpf_{name}")
        nws = 2 if RP_COMP else 1  # hi (+ lo) column partials
        self.ws_axpy = (ex.buf.alloc(max(8, nws * self.G * self.N * 8))
                        if self.axpy is not None else 0)
        self.ws_dot = ex.buf.alloc(max(8, self.ctiles * self.M * 8)) if self.dot is not None else 0

    # -- run ---------------------------------------------------------------------

    def _ptr(self, ex, view):
        return ex.buf.ptr[view.container] + 8 * view.offset

    def run(self, ex, sym, counters):
        cont, off = self.R[0], self.R[1]
        w = [0] * 8
        w[0] = ex.buf.ptr[cont] + 8 * off
        w[1] = self.ws_axpy
        w[2] = self.ws_dot
        if self.dot is not None:
            w[3] = self._ptr(ex, self.dot.vec)
            w[4] = self._ptr(ex, self.dot.out)
        if self.axpy is not None:
            if not self.coef_from_dot:
                w[5] = self._ptr(ex, self.axpy.vec)
            w[6] = self._ptr(ex, self.axpy.out)
        for d in self.pro_args:
            if d[0] == "ptr":
                w.append(ex.buf.ptr[d[1]])
            elif d[0] == "flag":
                w.append(ex.flag)
            else:
                raise P.PlanError(f"unsupported prologue argument {d}")
        blob = struct.pack(f"<{len(w)}q", *w)
        prof = ex._prof
        if prof is not None:
            ev = ex._prof_event_pair()
            ex._prof_record(ev[0])
        rt.launch(self.kmain, (self.G, self.ctiles, 1), (self.tpb, 1, 1), blob, ex.stream,
                  self.smem)
        if prof is not None:
            ex._prof_record(ev[1])
            prof.append((self.kmain.name, self.M * self.N, ev))
        nfin = max(self.N if self.axpy is not None else 0,
                   self.M if (self.dot is not None and self.ctiles > 1) else 0)
        if nfin:
            if prof is not None:
                ev = ex._prof_event_pair()
                ex._prof_record(ev[0])
            rt.launch(self.kfin, ((nfin + 31) // 32, 1, 1), (32, 32, 1), blob, ex.stream)
            if prof is not None:
                ex._prof_record(ev[1])
                prof.append((self.kfin.name, nfin, ev))
            ex.launches += 1
        ex.launches += 1
        if counters is not None:
            self._count(ex, sym, counters)

    def _count(self, ex, sym, counters):
        from .machine import _count_map

        if self.prologue is not None:
            rv = codegen.range_values(self.prologue, sym)
            _count_map(ex, self.prologue, rv, counters, sym)
        for mv in self.mvs:
            M, N = self.M, self.N
            counters.bytes_moved += 8 * (M * N + mv.vec.dims[0][0] + mv.out.dims[0][0])
            if mv.out_wcr is not None:
                counters.wcr_commits += mv.out.dims[0][0]


_ = ctypes
