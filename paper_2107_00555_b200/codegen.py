"""CUDA C generation for map groups (the generic map-scope kernel family).

A (fused) map group becomes one ``__global__`` kernel whose per-point body is
the scope's tasklet chain in the reference's execution order
(``Machine.exec_map`` runs children in topological order per point,
interp.py:420-441; ``exec_tasklet`` interp.py:400-418).  Memlet reads/writes
(interp.py:300-324) become loads/stores at row-major offsets; WCR writes
(ir.py:72-91) become plain read-modify-writes on thread-private locations and
atomics on shared ones; nested maps become in-thread loops; transients placed
in registers or per-thread scratch by the planner never touch HBM.

Thread mappings (chosen at plan time):
  scalar - one thread (top-level tasklets, fused in program order)
  seq    - one thread running the map lexicographically (SEQUENTIAL schedule)
  flat   - 1-D grid-stride over the flattened iteration space
  tile2  - 32x8 thread tiles over the two innermost parameters (coalesced
           along the last one), outer parameters flattened into the block
           index; virtual blocks are walked in order so concurrently resident
           CTAs touch neighbouring planes (L2 reuse for stencils)
"""

from __future__ import annotations

import math
import os
import re
import struct

from . import plan as P  # noqa: E402
from . import scalar, sdfg, symexpr

CT = {"f64": "double", "i64": "b2_ll", "i32": "int", "bool": "bool"}
TC = {"f64": "f", "i64": "i", "i32": "i", "bool": "b"}

MAX_BLOCKS = 148 * 16
HOIST_TILES = os.environ.get("B2_HOIST_TILES", "1") == "1"  # ... in flat / tile2 modes
REDUCE_MODE = os.environ.get("B2_REDUCE", "1") == "1"  # register-accumulated WCR reductions
# branch-free unrolled copy of the per-thread point loop for full tiles
MARCH_FULL = os.environ.get("B2_FULL_TILES", "1") == "1"
ROWRED_MODE = os.environ.get("B2_ROWRED", "1") == "1"  # warp-per-row WCR reductions
ROWRED_CONTIG = os.environ.get("B2_ROWRED_CONTIG", "1") == "1"  # pure reductions over the contiguous dim: rowred over reduce
ROWRED_CONTIG_MINROWS = 148 * 16  # ... when there are rows (warps) enough to fill the GPU
# the next map of a row reduction fused as its epilogue (softmax: ex / sm)
ROWRED_EPILOGUE = os.environ.get("B2_ROWRED_EPILOGUE", "1") == "1"
ROWRED_EPI_MINB = int(os.environ.get("B2_ROWRED_EPI_MINB", "3"))  # softmax 1.231 ms (2: 1.391, 4: 1.314, 8: spills)
FOLD_MODE = os.environ.get("B2_FOLD", "1") == "1"  # warp-cooperative max/min loop folds
SMALL_PRIVATE = 16  # elements: thread-private transients up to this size stay in registers
FOLD_UNROLL = int(os.environ.get("B2_FOLD_UNROLL", "4"))
TILE_BY = int(os.environ.get("B2_TILE_BY", "8"))  # tile rows (blockDim.y) in tile2 mode
MARCH_BY = int(os.environ.get("B2_MARCH_BY", "8"))  # tile rows (blockDim.y) in march mode
MARCH_BX = int(os.environ.get("B2_MARCH_BX", "64"))  # tile columns (blockDim.x) in march mode
# shift the innermost tile origin down to a 128-byte line so a warp's row
# access covers whole lines (march / tile2 with a constant unit-stride range)
RED_THREADS = int(os.environ.get("B2_RED_THREADS", str(148 * 8192)))  # chunked-reduction thread target (azimint 0.78 -> 0.51 ms vs 148 * 512)
RED_OUT_BLOCK = int(os.environ.get("B2_RED_OUT_BLOCK", "4"))  # outputs per thread, broadcast-read chunked reductions
SMALL_RED_CHUNK = int(os.environ.get("B2_SMALL_RED_CHUNK", "2"))  # terms per chunk, small reductions (0: off)
RED_BLOCK = int(os.environ.get("B2_RED_BLOCK", "16"))  # max points of a register-blocked output dim
MARCH_PREFETCH = os.environ.get("B2_MARCH_PF", "1") == "1"  # L2 bulk prefetch of march tiles
MARCH_PDL = os.environ.get("B2_MARCH_PDL", "1") == "1"  # march sweeps as programmatic dependent launches (heat 37.40 -> 37.24 ms)
# ... small flat / reduce / scalar kernels, whose launch latency is a large
# share of their time (nbody's per-step kernels: 5.32 -> 4.67 ms)
SMALL_PDL = os.environ.get("B2_SMALL_PDL", "1") == "1"
SMALL_PDL_POINTS = 1 << 16
# 2-D sweeps small enough to stay mostly in L2 (<= 2^24 points): each thread
# walks MARCH2_V consecutive rows of a 64-column tile and reuses the
# north / centre rows from registers (scripts/heatlab/jaclab.cu: jacobi_2d
# N=2000 8.03 vs 8.54 us per sweep for tile2; in the program with
# programmatic dependent launch 1.572 ms vs 1.735 for tile2, 1.670 without PDL)
MARCH2 = os.environ.get("B2_MARCH2", "1") == "1"
MARCH2_V = int(os.environ.get("B2_MARCH2_V", "16"))
MARCH2_BY = int(os.environ.get("B2_MARCH2_BY", "2"))  # 1.550 ms vs 1.57 at 4, 2.01 at 1
MARCH2_PDL = os.environ.get("B2_MARCH2_PDL", "1") == "1"
TILE_PDL = os.environ.get("B2_TILE_PDL", "0") == "1"  # ... tile2 sweeps (jacobi 1.74 -> 1.86 ms: off)
SLAB_PREFETCH = os.environ.get("B2_SLAB_PF", "1") == "1"  # ... in slab (runtime dim-0) sweeps
SLAB_BX = int(os.environ.get("B2_SLAB_BX", "32"))  # tile columns of slab sweeps
ROWRED_UNROLL = int(os.environ.get("B2_ROWRED_UNROLL", "1"))  # unroll of the warp-per-row loop (4 spilled at 32 regs)
ROWRED_MINB = int(os.environ.get("B2_ROWRED_MINB", "8"))  # min CTAs/SM for rowred kernels (softmax 1.11 -> 1.06 ms)
# row reductions: lane 0 L2-prefetches the warp's NEXT row of each read-only
# input while the current row is reduced (cp.async.bulk.prefetch.L2):
# softmax's row kernel 876 -> 836 us; GEMV row dots unchanged
ROWRED_PF = os.environ.get("B2_ROWRED_PF", "1") == "1"
SLAB_VEC = int(os.environ.get("B2_SLAB_VEC", "8"))  # planes per thread, runtime dim-0 range
# out[m, n] += X[m, k] * Y[k, n] maps (affine gathers, e.g. conv2d's 7-D WCR
# map) as an implicit GEMM on the FP64 tensor path (DMMA)
CONTRACT_MODE = os.environ.get("B2_CONTRACT", "1") == "1"
CONTRACT_MIN_FMA = 1 << 22
# m16 fragments per warp (CTA tile TM = 128 MF rows): conv2d_bias 0.760 ms at
# MF = 1, 0.705 at 2 (each B fragment feeds two DMMAs); BK = 32 is slower
CONTRACT_MF = int(os.environ.get("B2_CONTRACT_MF", "2"))
CONTRACT_BK = int(os.environ.get("B2_CONTRACT_BK", "16"))  # k chunk staged per barrier
# contractions whose X operand slides along the fastest output parameter
# (convolutions: X[n, i + ki, j + kj, ci]): stage one contiguous window of X
# per (tile, k chunk) instead of gathering every (row, k) element
CONTRACT_SLIDE = os.environ.get("B2_CONTRACT_SLIDE", "1") == "1"
CONTRACT_SLIDE_MAXWIN = 4096  # doubles per window buffer
CONTRACT_SLIDE_BK = int(os.environ.get("B2_CONTRACT_SLIDE_BK", "0"))  # 0: largest k chunk <= 64 dividing the run
# 3-D stencil sweeps through a TMA plane ring (cp.async.bulk.tensor.3d into
# shared memory, mbarrier-tracked, persistent balanced grid): the tma3 mode
# (measured: heat_3d N=400 39.3 ms vs 37.3 for march at the best geometry
# below — bitwise equal, not the default)
TMA3 = os.environ.get("B2_TMA3", "0") == "1"
TMA3_CTAS = int(os.environ.get("B2_TMA3_CTAS", "1"))  # resident CTAs per SM (grid = 148 x this)
TMA3_PREF = int(os.environ.get("B2_TMA3_PREF", "2"))  # planes in flight beyond the stencil window
TMA3_TJ = int(os.environ.get("B2_TMA3_TJ", "16"))  # tile rows (a multiple of the consumer warps)
TMA3_L2PF = int(os.environ.get("B2_TMA3_L2PF", "0"))  # planes L2-prefetched ahead of the ring
TMA3_CHUNK = int(os.environ.get("B2_TMA3_CHUNK", "32"))  # planes per CTA (0: persistent balanced grid)
TMA3_CW = int(os.environ.get("B2_TMA3_CW", "8"))  # consumer warps per CTA (+1 producer warp)


class KernelSpec:
    """Generated kernel + host-side launch recipe."""

    def __init__(self):
        self.name = ""
        self.source = ""
        self.mode = "flat"
        self.block = (256, 1, 1)
        self.args: list[tuple] = []  # arg descriptors, in blob order
        self.syms: list[str] = []
        self.containers: list[str] = []
        self.private: dict[str, int] = {}  # container -> elements per thread
        self.checks: list[tuple] = []  # (container, subset, rename) depth-0 memory accesses
        self.sites: list[str] = []  # device OOB guard site descriptions
        self.uses_flag = False
        self.params: list[str] = []
        self.vec = 1
        self.dyn0 = False  # range of the first parameter is a runtime argument
        self.align = 0  # elements the innermost tile origin is shifted down by
        self.kernel = None  # runtime.Kernel
        self.tmaps: list[tuple] = []  # (container, box (inner..outer)) TMA maps ahead of the args
        self.smem = 0  # dynamic shared memory bytes
        self.grid_cap = 0  # tma3: persistent grid size
        self.epilogue = None  # index of the map group run as this kernel's epilogue

    def arg_index(self, desc) -> int:
        try:
            return self.args.index(desc)
        except ValueError:
            self.args.append(desc)
            return len(self.args) - 1


class _Gen:
    def __init__(self, planner: P.Planner, group: P.MapGroup, shapes: dict, name: str):
        self.pl = planner
        self.g = planner.g
        self.group = group
        self.shapes = shapes
        self.spec = KernelSpec()
        self.spec.name = name
        self.lines: list[str] = []
        self.uid = 0
        self.regs: list[str] = []
        self.ind = 2
        self.arg_base = 0
        self.place_override: dict[str, str] = {}
        self.written: set = set()
        self.cse: dict = {}
        self.stencil: dict = {}
        self.hoist = False
        self.hoisted: list = []
        self.colstage: dict = {}
        self.red = None  # reduction mode: target key -> accumulator info
        self.red_targets: dict = {}
        self.red_pout: list = []
        self.red_full = False
        self.ptr_override: dict[str, str] = {}  # container -> C pointer name
        self.init_const: dict[str, str] = {}  # reduction target -> fused init constant
        self.read_set: set = set()
        self.redirect: dict[str, str] = {}  # container -> C expression (register copies)
        self.epi_group = None  # a map fused as the epilogue of a row reduction
        self.epi = None
        self.rowred_pointw: dict = {}

    def _wkey(self, m: sdfg.Memlet, env: dict):
        rename = {mp: v[2:] for mp, v in env.items() if isinstance(v, str) and v.startswith("p_")}
        keys = tuple(self.group.params) + tuple(sorted(self.pl.loopish))
        return (m.container, tuple(P.canon(P.rn(b, rename), keys, self.pl.fixed)
                                   for b, _, _ in m.subset))

    def _old(self, t) -> str:
        """The value a reduction target holds before this kernel: memory, or
        the constant the executor's fused init map would have stored."""
        lit = self.init_const.get(t.get("cont"))
        return f"(({t['ct']})({lit}))" if lit is not None else t["target"]

    def _contraction_plan(self):
        """``O[m(p), n] (+)= X[a(p)] * Y[b(p)]``: one scope, one tasklet that
        is the product of its two inputs, a WCR-add output indexed by one
        parameter per dimension (the output parameters), X and Y affine in
        the parameters.  The output parameter that only Y uses is the GEMM's
        N; the other output parameters (used by X, not by Y) are M; the rest
        are K.  Returns the address coefficients or None."""
        grp = self.group
        if grp.schedule != "parallel" or len(grp.members) != 1:
            return None
        if any(r is None or r[2] < 1 for r in self.const_ranges):
            return None
        mem = grp.members[0]
        kids = ([mem.tasklet] if mem.tasklet is not None else
                list(P._scope_children(mem.state, mem.entry)))
        nested = [k for k in kids if not isinstance(k, sdfg.MapExit)]
        if len(nested) == 1 and isinstance(nested[0], sdfg.MapEntry):
            return self._blocked_contraction_plan(mem, nested[0])
        ents = [k for k in nested if isinstance(k, sdfg.MapEntry)]
        libs = [k for k in nested if isinstance(k, sdfg.Library)]
        if len(ents) == 1 and len(libs) == 1 and all(
                isinstance(k, (sdfg.MapEntry, sdfg.Library, sdfg.Access)) for k in nested):
            return self._mapreduce_contraction_plan(mem, ents[0], libs[0])
        tks = [k for k in nested if isinstance(k, sdfg.Tasklet)]
        if len(ents) == 2 and not libs and len(tks) == 1 and all(
                isinstance(k, (sdfg.MapEntry, sdfg.Tasklet, sdfg.Access)) for k in nested):
            tiled = self._tiled_sum_match(mem, ents, tks[0])
            if tiled is not None:
                return self._mapreduce_contraction_plan(mem, tiled["producer"], None, tiled)
        if len(kids) != 1 or not isinstance(kids[0], sdfg.Tasklet):
            return None
        t = kids[0]
        if len(t.code) != 1 or len(t.ins) != 2:
            return None
        code = t.code[0][1]
        if code[0] != "bin" or code[1] != "*" or {code[2], code[3]} != \
                {("ref", t.ins[0]), ("ref", t.ins[1])}:
            return None
        ins = {e.dst_conn: e.memlet for e in mem.state.in_edges(t) if e.memlet is not None}
        outs = [e.memlet for e in mem.state.out_edges(t) if e.memlet is not None]
        if len(outs) != 1 or outs[0].wcr != "add" or set(ins) != set(t.ins):
            return None
        acc = {(c, w): (wcr, depth, pt)
               for (c, w, wcr, depth, pt) in self.pl.member_accesses(mem, grp.params)}
        if len(acc) != 3:
            return None
        params = list(grp.params)

        def coeffs(cont, pt):
            if pt is None or self.place(cont) != "memory" or self.g.containers[cont].dtype != "f64":
                return None
            st = _row_major(self.shapes[cont])
            if len(pt) != len(st):
                return None
            cst, co = 0, {}
            for d, (c0, terms) in enumerate(pt):
                cst += st[d] * c0
                for q, cq in terms:
                    co[q] = co.get(q, 0) + st[d] * cq
            return cst, co

        oc = outs[0].container
        wcr, depth, opt = acc.get((oc, True), (None, 1, None))
        if wcr != "add" or depth != 0 or opt is None:
            return None
        xs = [ins[c].container for c in t.ins]
        if len(set(xs)) != 2 or oc in xs:
            return None
        ca = [coeffs(c, acc[(c, False)][2]) for c in xs]
        co_ = coeffs(oc, opt)
        if None in ca or co_ is None or any(acc[(c, False)][1] != 0 for c in xs):
            return None
        pout = []
        for c0, terms in opt:
            if len(terms) != 1 or terms[0][1] != 1:
                return None
            pout.append(terms[0][0])
        if len(set(pout)) != len(pout):
            return None
        used = [set(q for q, v in c[1].items() if v) for c in ca]
        outs_ = [set(pout) & u for u in used]
        if outs_[0] & outs_[1] or (outs_[0] | outs_[1]) != set(pout):
            return None
        # the operand indexed by a single output parameter carries N
        yi = 1 if len(outs_[1]) == 1 else (0 if len(outs_[0]) == 1 else None)
        if yi is None:
            return None
        xi = 1 - yi
        npar = next(iter(outs_[yi]))
        M = [q for q in params if q in pout and q != npar]
        K = [q for q in params if q not in pout]
        if not M or not K or any(q in used[yi] for q in M):
            return None
        ext = {q: self.const_ranges[params.index(q)][2] for q in params}
        fma = 1
        for q in params:
            fma *= ext[q]
        if fma < CONTRACT_MIN_FMA:
            return None
        return {"X": xs[xi], "Y": xs[yi], "O": oc, "cx": ca[xi], "cy": ca[yi], "co": co_,
                "M": M, "N": npar, "K": K, "ext": ext,
                "rng": {q: self.const_ranges[params.index(q)] for q in params}}

    def _tiled_sum_match(self, mem, ents, zero):
        """auto_optimize's tiled REDUCE expansion inside a map (tile_wcr,
        autoopt.py:480-595; doitgen.auto): ``O = 0``, then per tile
        ``acc = 0; acc += T[k]`` over the tile's k (sequential), ``O += acc``
        (WCR add), the tiles partitioning T's range.  Returns the producer
        map of T and the O edges, or None."""
        st = mem.state

        def kids(e):
            return [k for k in P._scope_children(st, e) if not isinstance(k, sdfg.MapExit)]

        def only_code(t):
            return t.code[0][1] if len(t.code) == 1 else None

        zo = [e for e in st.out_edges(zero) if e.memlet is not None]
        if zero.ins or len(zo) != 1 or zo[0].memlet.wcr is not None or \
                only_code(zero) not in (("num", 0.0), ("num", 0)):
            return None
        O = zo[0].memlet
        for prod, tile in (ents, ents[::-1]):
            pk = [k for k in kids(prod)]
            tk = kids(tile)
            if len(pk) != 1 or not isinstance(pk[0], sdfg.Tasklet) or len(tile.params) != 1:
                continue
            pouts = [e for e in st.out_edges(pk[0]) if e.memlet is not None]
            if len(pouts) != 1:
                continue
            T = pouts[0].memlet.container
            inner = [k for k in tk if isinstance(k, sdfg.MapEntry)]
            tts = [k for k in tk if isinstance(k, sdfg.Tasklet)]
            if len(inner) != 1 or len(tts) != 2 or len(inner[0].params) != 1 \
                    or any(not isinstance(k, (sdfg.MapEntry, sdfg.Tasklet, sdfg.Access)) for k in tk):
                continue
            red = kids(inner[0])
            if len(red) != 1 or not isinstance(red[0], sdfg.Tasklet):
                continue
            rt_ = red[0]
            rin = {e.dst_conn: e.memlet for e in st.in_edges(rt_) if e.memlet is not None}
            rout = [e.memlet for e in st.out_edges(rt_) if e.memlet is not None]
            code = only_code(rt_)
            if not (len(rin) == 2 and len(rout) == 1 and code is not None and code[0] == "bin"
                    and code[1] == "+"):
                continue
            accn = rout[0].container
            tin = [c for c, m in rin.items() if m.container == T]
            ain = [c for c, m in rin.items() if m.container == accn]
            if len(tin) != 1 or len(ain) != 1 or \
                    {code[2], code[3]} != {("ref", tin[0]), ("ref", ain[0])}:
                continue
            kq = inner[0].params[0][0]
            if rin[tin[0]].subset[0][:2] != (("s", kq), ("s", kq)) and \
                    tuple(rin[tin[0]].subset[0][:2]) != (("s", kq), ("s", kq)):
                continue
            init = [t for t in tts if t is not rt_ and not t.ins]
            fin = [t for t in tts if t is not rt_ and t.ins]
            if len(init) != 1 or len(fin) != 1 or only_code(init[0]) not in (("num", 0.0), ("num", 0)):
                continue
            io = [e for e in st.out_edges(init[0]) if e.memlet is not None]
            fo = [e for e in st.out_edges(fin[0]) if e.memlet is not None]
            fi = [e for e in st.in_edges(fin[0]) if e.memlet is not None]
            if len(io) != 1 or io[0].memlet.container != accn or len(fo) != 1 or len(fi) != 1 \
                    or fi[0].memlet.container != accn or fo[0].memlet.wcr != "add" \
                    or fo[0].memlet.text != O.text or only_code(fin[0]) != ("ref", fin[0].ins[0]):
                continue
            # the tiles' k ranges partition T (numerically, at the bound sizes)
            env = dict(self.pl.fixed)
            tp, (tb, te, ts) = tile.params[0]
            try:
                tvals = range(symexpr.evaluate(tb, env), symexpr.evaluate(te, env) + 1,
                              symexpr.evaluate(ts, env))
                seen = []
                for v in tvals:
                    e2 = dict(env)
                    e2[tp] = v
                    b, e, s_ = (symexpr.evaluate(x, e2) for x in inner[0].params[0][1])
                    seen.extend(range(b, e + 1, s_))
            except Exception:
                continue
            if seen != list(range(self.shapes[T][0])):
                continue
            return {"producer": prod, "T": T, "o_edge": fo[0], "zero_edge": zo[0]}
        return None

    def _mapreduce_contraction_plan(self, mem, inner, lib, tiled=None):
        """``out[m, n] = sum(T)`` after ``T[k] = X[m, k] * Y[k, n]`` inside
        one parallel map (doitgen's pipe / LoopToMap form: a map into a
        transient row, then a whole-array REDUCE): per output point the sum
        over k of the flat product, so the contraction kernel computes it
        with its accumulators starting from zero (O is overwritten) and T is
        never materialised.  Re-associated like every tensor-core product
        (within the rel_err 1e-12 contract)."""
        st = mem.state
        grp = self.group
        if tiled is not None:
            T = tiled["T"]
            lout = [tiled["o_edge"]]
            lin = None
        else:
            if lib.kind != "reduce" or lib.attrs.get("axes") is not None \
                    or lib.attrs.get("op", "add") != "add":
                return None
            lin = [e for e in st.in_edges(lib) if e.memlet is not None]
            lout = [e for e in st.out_edges(lib) if e.memlet is not None]
            if len(lin) != 1 or len(lout) != 1 or lout[0].memlet.wcr is not None:
                return None
            T = lin[0].memlet.container
        tc = self.g.containers[T]
        if not tc.transient or len(self.shapes[T]) != 1:
            return None
        if {s_.op for s_ in self.pl.sites.get(T, [])} != {grp.idx}:
            return None  # T read elsewhere: it must be materialised
        kids = [k for k in P._scope_children(st, inner) if not isinstance(k, sdfg.MapExit)]
        if len(kids) != 1 or not isinstance(kids[0], sdfg.Tasklet) or len(inner.params) != 1:
            return None
        t = kids[0]
        if len(t.code) != 1 or len(t.ins) != 2:
            return None
        code = t.code[0][1]
        if code[0] != "bin" or code[1] != "*" or {code[2], code[3]} != \
                {("ref", t.ins[0]), ("ref", t.ins[1])}:
            return None
        ins = {e.dst_conn: e.memlet for e in st.in_edges(t) if e.memlet is not None}
        touts = [e.memlet for e in st.out_edges(t) if e.memlet is not None]
        kp, (kb, ke, ks) = inner.params[0]
        if len(touts) != 1 or touts[0].container != T or touts[0].wcr is not None:
            return None
        if touts[0].subset != [(("s", kp), ("s", kp), ("c", 1))] and \
                tuple(tuple(x) for x in touts[0].subset[0][:2]) != (("s", kp), ("s", kp)):
            return None
        kr = _const_range(self.pl, (kb, ke, ks))
        if kr is None or kr != (0, 1, self.shapes[T][0]):
            return None  # T[k] over the whole of T, k ascending
        if lin is not None and _const_range(self.pl, lin[0].memlet.subset[0]) != \
                (0, 1, self.shapes[T][0]):
            return None
        params = list(grp.params) + [kp]
        if kp in grp.params:
            return None
        env = dict(self.pl.fixed)

        def pt_of(m):
            out = []
            for (b, e, s_) in m.subset:
                if b != e:
                    return None
                a = symexpr.affine(b, tuple(params), env)
                if a is None:
                    return None
                out.append((a[0], tuple(sorted(a[1].items()))))
            return tuple(out)

        def coeffs(cont, pt):
            if pt is None or self.place(cont) != "memory" or self.g.containers[cont].dtype != "f64":
                return None
            st_ = _row_major(self.shapes[cont])
            if len(pt) != len(st_):
                return None
            cst, co = 0, {}
            for d, (c0, terms) in enumerate(pt):
                cst += st_[d] * c0
                for q, cq in terms:
                    co[q] = co.get(q, 0) + st_[d] * cq
            return cst, co

        oc = lout[0].memlet.container
        xs = [ins[c].container for c in t.ins]
        if len(set(xs)) != 2 or oc in xs or T in xs:
            return None
        opt = pt_of(lout[0].memlet)
        ca = [coeffs(c, pt_of(ins[conn])) for c, conn in zip(xs, t.ins)]
        co_ = coeffs(oc, opt)
        if None in ca or co_ is None or opt is None:
            return None
        pout = []
        for c0, terms in opt:
            if len(terms) != 1 or terms[0][1] != 1:
                return None
            pout.append(terms[0][0])
        if len(set(pout)) != len(pout) or set(pout) != set(grp.params):
            return None
        used = [set(q for q, v in c[1].items() if v) for c in ca]
        outs_ = [set(pout) & u for u in used]
        if outs_[0] & outs_[1] or (outs_[0] | outs_[1]) != set(pout):
            return None
        yi = 1 if len(outs_[1]) == 1 else (0 if len(outs_[0]) == 1 else None)
        if yi is None:
            return None
        xi = 1 - yi
        npar = next(iter(outs_[yi]))
        M = [q for q in grp.params if q != npar]
        K = [kp]
        if not M or any(q in used[yi] for q in M):
            return None
        rng = {q: self.const_ranges[grp.params.index(q)] for q in grp.params}
        rng[kp] = kr
        if any(r is None for r in rng.values()):
            return None
        ext = {q: rng[q][2] for q in params}
        fma = 1
        for q in params:
            fma *= ext[q]
        if fma < CONTRACT_MIN_FMA:
            return None
        return {"X": xs[xi], "Y": xs[yi], "O": oc, "cx": ca[xi], "cy": ca[yi], "co": co_,
                "M": M, "N": npar, "K": K, "ext": ext, "rng": rng, "init_zero": True,
                "checks": st.in_edges(inner) + lout + ([tiled["zero_edge"]] if tiled else [])}

    def _blocked_contraction_plan(self, mem, inner):
        """The reference's blocked MATMUL expansion (autoopt.py:707-813,
        ``blocked_native``): a PARALLEL map over output tiles (ib, jb) around
        one SEQUENTIAL map (i, j, k) whose i / j ranges are the tile's rows /
        columns and k the whole reduction, one tasklet ``a * b`` with a WCR
        add into O[i, j].  Per (i, j) that is the k-ascending sum of the
        flat product, so it runs as the same DMMA implicit GEMM over the
        flattened space (re-associated like every tensor-core product:
        within the rel_err 1e-12 contract).  The tiles must partition the
        output exactly (checked on the bound extents)."""
        st = mem.state
        grp = self.group
        kids = [k for k in P._scope_children(st, inner) if not isinstance(k, sdfg.MapExit)]
        if len(kids) != 1 or not isinstance(kids[0], sdfg.Tasklet) or inner.schedule == "parallel":
            return None
        t = kids[0]
        if len(t.code) != 1 or len(t.ins) != 2:
            return None
        code = t.code[0][1]
        if code[0] != "bin" or code[1] != "*" or {code[2], code[3]} != \
                {("ref", t.ins[0]), ("ref", t.ins[1])}:
            return None
        ins = {e.dst_conn: e.memlet for e in st.in_edges(t) if e.memlet is not None}
        outs = [e.memlet for e in st.out_edges(t) if e.memlet is not None]
        if len(outs) != 1 or outs[0].wcr != "add" or set(ins) != set(t.ins):
            return None
        env = dict(self.pl.fixed)
        outer = [mp for mp, gp in mem.rename.items()]  # member's own outer parameter names
        oranges = {mp: self.const_ranges[grp.params.index(gp)] for mp, gp in mem.rename.items()}
        iparams = inner.param_names
        # flattened extents: the union over the outer tiles of each inner range
        flat = {}
        for q, (b, e, s_) in inner.params:
            if symexpr.free_symbols(s_) - set(env) or symexpr.evaluate(s_, env) != 1:
                return None
            deps = (symexpr.free_symbols(b) | symexpr.free_symbols(e)) & set(outer)
            if len(deps) > 1:
                return None
            covered = []
            vals = [None]
            if deps:
                d = next(iter(deps))
                r0, r1, rn = oranges[d]
                vals = [(d, r0 + r1 * x) for x in range(rn)]
            for v in vals:
                ev = dict(env)
                if v is not None:
                    ev[v[0]] = v[1]
                try:
                    lo, hi = symexpr.evaluate(b, ev), symexpr.evaluate(e, ev)
                except KeyError:
                    return None
                if hi >= lo:
                    covered.append((lo, hi))
            covered.sort()
            pos = 0
            for lo, hi in covered:
                if lo != pos:
                    return None  # gaps or overlaps: not a partition
                pos = hi + 1
            if not covered or covered[0][0] != 0:
                return None
            flat[q] = (0, 1, pos)
        # the tiles must vary independently (every (ib, jb) pair present)
        if len({d for q, (b, e, s_) in inner.params
                for d in (symexpr.free_symbols(b) | symexpr.free_symbols(e)) & set(outer)}) \
                != len(outer):
            return None

        def pt_of(m):
            out = []
            for (b, e, s_) in m.subset:
                if b != e:
                    return None
                a = symexpr.affine(b, tuple(iparams), env)
                if a is None:
                    return None
                out.append((a[0], tuple(sorted(a[1].items()))))
            return tuple(out)

        def coeffs(cont, pt):
            if pt is None or self.place(cont) != "memory" or self.g.containers[cont].dtype != "f64":
                return None
            st_ = _row_major(self.shapes[cont])
            if len(pt) != len(st_):
                return None
            cst, co = 0, {}
            for d, (c0, terms) in enumerate(pt):
                cst += st_[d] * c0
                for q, cq in terms:
                    co[q] = co.get(q, 0) + st_[d] * cq
            return cst, co

        oc = outs[0].container
        xs = [ins[c].container for c in t.ins]
        if len(set(xs)) != 2 or oc in xs:
            return None
        opt = pt_of(outs[0])
        ca = [coeffs(c, pt_of(ins[conn])) for c, conn in zip(xs, t.ins)]
        co_ = coeffs(oc, opt)
        if None in ca or co_ is None or opt is None:
            return None
        pout = []
        for c0, terms in opt:
            if len(terms) != 1 or terms[0][1] != 1:
                return None
            pout.append(terms[0][0])
        if len(set(pout)) != len(pout):
            return None
        used = [set(q for q, v in c[1].items() if v) for c in ca]
        outs_ = [set(pout) & u for u in used]
        if outs_[0] & outs_[1] or (outs_[0] | outs_[1]) != set(pout):
            return None
        yi = 1 if len(outs_[1]) == 1 else (0 if len(outs_[0]) == 1 else None)
        if yi is None:
            return None
        xi = 1 - yi
        npar = next(iter(outs_[yi]))
        M = [q for q in iparams if q in pout and q != npar]
        K = [q for q in iparams if q not in pout]
        if not M or not K or any(q in used[yi] for q in M):
            return None
        ext = {q: flat[q][2] for q in iparams}
        fma = 1
        for q in iparams:
            fma *= ext[q]
        if fma < CONTRACT_MIN_FMA:
            return None
        return {"X": xs[xi], "Y": xs[yi], "O": oc, "cx": ca[xi], "cy": ca[yi], "co": co_,
                "M": M, "N": npar, "K": K, "ext": ext, "rng": flat}

    def _slide_plan(self, cp):
        """X's address is R(outer M) + S * j + kx(k) with j the fastest M
        parameter, and the fastest K parameters form a contiguous run of KR
        addresses (conv2d_bias: kx = 768 ki + 3 kj + ci, KR = 60).  With k
        chunks inside one run, the A tile of TM consecutive j's is the
        contiguous window X[R + S j0 + kx(k0) .. + S (TM - 1) + BK)."""
        Mp, Kp, ext, rng = cp["M"], cp["K"], cp["ext"], cp["rng"]
        cx = cp["cx"][1]
        jm = Mp[-1]
        S = cx.get(jm, 0) * rng[jm][1]
        if S <= 0:
            return None
        run = 1
        for q in reversed(Kp):
            c = cx.get(q, 0) * rng[q][1]
            if c != run:
                break
            run *= ext[q]
        order = (CONTRACT_SLIDE_BK,) if CONTRACT_SLIDE_BK else (64, 60, 56, 48, 40, 32, 24, 20, 16, 12, 8)
        BK = next((b for b in order if run % b == 0), None)
        if BK is None:
            return None
        TM = 128 * CONTRACT_MF
        WS = S * (TM - 1) + BK
        if WS > CONTRACT_SLIDE_MAXWIN:
            return None
        return {"S": S, "BK": BK, "KR": run, "WS": WS + (WS & 1), "jm": jm}

    def _contract_slide_kernel(self, cp, sl):
        """The contraction kernel with a sliding X window (see _slide_plan):
        M tiles are TM consecutive values of the fastest M parameter j within
        one outer point (rows past the last j compute garbage that is never
        stored), each k chunk stages X[R + S j0 + kx(k0) ...] (one coalesced
        contiguous range, register double-buffered) and the A fragments read
        it at S * row + k.  Same DMMA order as _contract_kernel: within 1e-12
        of the sequential reference sum, not bitwise."""
        spec = self.spec
        X, Y, O = cp["X"], cp["Y"], cp["O"]
        Mp, Kp, Np = cp["M"], cp["K"], cp["N"]
        ext, rng = cp["ext"], cp["rng"]
        decode = self._contract_decode(cp)
        Mtot = math.prod(ext[q] for q in Mp)
        Ktot = math.prod(ext[q] for q in Kp)
        Ntot = ext[Np]
        EJ = ext[sl["jm"]]
        TN = 8 * min(4, -(-Ntot // 8))
        NF = TN // 8
        MF, BK, S, WS = CONTRACT_MF, sl["BK"], sl["S"], sl["WS"]
        TM = 128 * MF
        ax, ay, ao = (self.arg(("ptr", X)), self.arg(("ptr", Y)), self.arg(("ptr", O)))
        for c in (X, Y, O):
            self.cont(c)
        cyn = cp["cy"][1].get(Np, 0)
        con = cp["co"][1].get(Np, 0)
        L = [f"// generated by paper_2107_00555_b200.codegen: sliding-window contraction "
             f"(DMMA implicit GEMM) M={Mtot} N={Ntot} K={Ktot} S={S} KR={sl['KR']}",
             "struct B2Args { long long w[%d]; };" % max(1, len(spec.args)),
             "namespace {",
             f"constexpr int MF = {MF}, TM = {TM}, BK = {BK}, TN = {TN}, NF = {NF}, BPAD = 4;",
             f"constexpr int S = {S}, WS = {WS}, WR = (WS + 255) / 256;",
             f"constexpr long long MT = {Mtot}LL, NT = {Ntot}LL, KT = {Ktot}LL, EJ = {EJ}LL;",
             "constexpr long long NJB = (EJ + TM - 1) / TM, MO = MT / EJ;",
             "__device__ __forceinline__ void b2c_dmma(double (&d)[4], double a0, double a1, "
             "double b0) {",
             '  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, '
             '{%4,%5}, {%6}, {%0,%1,%2,%3};\\n" : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) '
             ': "d"(a0), "d"(a1), "d"(b0));',
             "}",
             "__device__ __forceinline__ long long b2c_mx(unsigned m) { return "
             + decode(Mp, cp["cx"], "m") + "; }",
             "__device__ __forceinline__ long long b2c_kx(unsigned k) { return "
             + decode(Kp, cp["cx"], "k") + "; }",
             "__device__ __forceinline__ long long b2c_ky(unsigned k) { return "
             + decode(Kp, cp["cy"], "k") + "; }",
             "__device__ __forceinline__ long long b2c_mo(unsigned m) { return "
             + decode(Mp, cp["co"], "m") + "; }",
             "}  // namespace",
             f'extern "C" __global__ void __launch_bounds__(256) {spec.name}'
             f"(const __grid_constant__ B2Args a) {{",
             "  B2_PDL_ENTRY();",
             f"  const double *__restrict__ X = (const double *){ax} + {cp['cx'][0]}LL;",
             f"  const double *__restrict__ Y = (const double *){ay} + {cp['cy'][0]}LL;",
             f"  double *__restrict__ O = (double *){ao} + {cp['co'][0]}LL;",
             "  extern __shared__ __align__(16) double b2c_smem[];",
             "  double (*Win)[WS] = reinterpret_cast<double (*)[WS]>(b2c_smem);",
             "  double (*Bs)[BK][TN + BPAD] = reinterpret_cast<double (*)[BK][TN + BPAD]>("
             "b2c_smem + 2 * WS);",
             "  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;",
             "  const int g = lane >> 2, t = lane & 3;",
             "  const long long ntiles = (NT + TN - 1) / TN;",
             "  for (long long tile = blockIdx.x; tile < MO * NJB * ntiles; tile += gridDim.x) {",
             "    const long long tm = tile / ntiles, n0 = (tile % ntiles) * TN;",
             "    const long long j0 = (tm % NJB) * TM, mfirst = (tm / NJB) * EJ + j0;",
             "    const long long rows = EJ - j0 < TM ? EJ - j0 : TM;",
             "    const long long R = b2c_mx((unsigned)mfirst);",
             "    const int wl = (int)(S * (rows - 1) + BK);",
             "    double rw[WR], rb[(BK * TN + 255) / 256];",
             "    auto load = [&](long long k0) {",
             "      const double *src = X + R + b2c_kx((unsigned)k0);",
             "#pragma unroll",
             "      for (int r = 0; r < WR; ++r) {",
             "        const int e = tid + 256 * r;",
             "        rw[r] = e < wl ? src[e] : 0.0;",
             "      }",
             "#pragma unroll",
             "      for (int r = 0; r < (BK * TN + 255) / 256; ++r) {",
             "        const int e = tid + 256 * r;",
             "        if (e < BK * TN) {",
             "          const int row = e / TN, col = e % TN;",
             "          const long long k = k0 + row, n = n0 + col;",
             f"          rb[r] = n < NT ? Y[b2c_ky((unsigned)k) + {cyn}LL * "
             f"({rng[Np][0]}LL + {rng[Np][1]}LL * n)] : 0.0;",
             "        }",
             "      }",
             "    };",
             "    auto store = [&](int buf) {",
             "#pragma unroll",
             "      for (int r = 0; r < WR; ++r) {",
             "        const int e = tid + 256 * r;",
             "        if (e < WS) Win[buf][e] = rw[r];",
             "      }",
             "#pragma unroll",
             "      for (int r = 0; r < (BK * TN + 255) / 256; ++r) {",
             "        const int e = tid + 256 * r;",
             "        if (e < BK * TN) Bs[buf][e / TN][e % TN] = rb[r];",
             "      }",
             "    };",
             "    double acc[MF][NF][4];",
             "    const int wm = warp * 16 * MF;",
             "#pragma unroll",
             "    for (int mf = 0; mf < MF; ++mf)",
             "#pragma unroll",
             "    for (int f = 0; f < NF; ++f)",
             "#pragma unroll",
             "      for (int h = 0; h < 2; ++h)",
             "#pragma unroll",
             "        for (int e2 = 0; e2 < 2; ++e2) {",
             "          const int row = wm + 16 * mf + g + 8 * h;",
             "          const long long n = n0 + f * 8 + 2 * t + e2;",
             ("          acc[mf][f][2 * h + e2] = 0.0; (void)row; (void)n;" if cp.get("init_zero") else
              f"          acc[mf][f][2 * h + e2] = (row < rows && n < NT) ? "
              f"O[b2c_mo((unsigned)(mfirst + row)) + {con}LL * "
              f"({rng[Np][0]}LL + {rng[Np][1]}LL * n)] : 0.0;"),
             "        }",
             "    __syncthreads();",
             "    load(0);",
             "    store(0);",
             "    __syncthreads();",
             "    const long long nk = KT / BK;",
             "    for (long long kc = 0; kc < nk; ++kc) {",
             "      const int cur = (int)(kc & 1);",
             "      if (kc + 1 < nk) load((kc + 1) * BK);",
             "      const double *win = Win[cur];",
             "#pragma unroll",
             "      for (int k4 = 0; k4 < BK; k4 += 4) {",
             "        double bf[NF];",
             "#pragma unroll",
             "        for (int f = 0; f < NF; ++f) bf[f] = Bs[cur][k4 + t][f * 8 + g];",
             "#pragma unroll",
             "        for (int mf = 0; mf < MF; ++mf) {",
             "          if (wm + 16 * mf >= rows) break;  // m16 fragment past the row's last j",
             "          const int r0 = wm + 16 * mf + g;",
             "          const double a0 = win[S * r0 + k4 + t], a1 = win[S * (r0 + 8) + k4 + t];",
             "#pragma unroll",
             "          for (int f = 0; f < NF; ++f) b2c_dmma(acc[mf][f], a0, a1, bf[f]);",
             "        }",
             "      }",
             "      if (kc + 1 < nk) store(cur ^ 1);",
             "      __syncthreads();",
             "    }",
             "#pragma unroll",
             "    for (int mf = 0; mf < MF; ++mf)",
             "#pragma unroll",
             "    for (int f = 0; f < NF; ++f)",
             "#pragma unroll",
             "      for (int h = 0; h < 2; ++h)",
             "#pragma unroll",
             "        for (int e2 = 0; e2 < 2; ++e2) {",
             "          const int row = wm + 16 * mf + g + 8 * h;",
             "          const long long n = n0 + f * 8 + 2 * t + e2;",
             f"          if (row < rows && n < NT) O[b2c_mo((unsigned)(mfirst + row)) + {con}LL * "
             f"({rng[Np][0]}LL + {rng[Np][1]}LL * n)] = acc[mf][f][2 * h + e2];",
             "        }",
             "  }",
             "}"]
        self._contract_checks(cp)
        spec.source = "\n".join(L) + "\n"
        spec.block = (256, 1, 1)
        spec.vec = 1
        spec.pdl = False
        spec.contract = {"M": Mtot, "N": Ntot, "K": Ktot, "TN": TN, "TM": TM,
                         "tiles_m": (Mtot // EJ) * (-(-EJ // TM)), "slide": dict(sl)}
        spec.smem = 8 * (2 * WS + 2 * BK * (TN + 4))
        return spec

    def _contract_decode(self, cp):
        ext, rng = cp["ext"], cp["rng"]

        def decode(names, cst_co, idx):
            """C expression: address part of a flat index over ``names``
            (mixed radix, last name fastest)."""
            _, co = cst_co
            rem = idx
            out = []
            for i, q in enumerate(reversed(names)):
                e = ext[q]
                v = f"(({rem}) % {e}u)" if i < len(names) - 1 else f"({rem})"
                rem = f"(({rem}) / {e}u)"
                val = f"({rng[q][0]}LL + {rng[q][1]}LL * (long long){v})"
                c = co.get(q, 0)
                if c:
                    out.append(f"{c}LL * {val}")
            return " + ".join(out) if out else "0LL"
        return decode

    def _contract_checks(self, cp=None):
        """Host-side bounds checks of the three memlets (as the generic
        body's)."""
        spec = self.spec
        mem = self.group.members[0]
        menv = {mp: f"p_{gp}" for mp, gp in mem.rename.items()}
        if cp is not None and cp.get("checks") is not None:
            for e in cp["checks"]:
                if e.memlet is not None:
                    spec.checks.append((e.memlet.container, e.memlet.subset, menv))
            return
        t = next(k for k in P._scope_children(mem.state, mem.entry)
                 if not isinstance(k, sdfg.MapExit)) if mem.tasklet is None else mem.tasklet
        if isinstance(t, sdfg.MapEntry):  # blocked form: the inner map's outer memlets
            edges = mem.state.in_edges(t) + mem.state.out_edges(mem.state.exit_of(t))
        else:
            edges = mem.state.in_edges(t) + mem.state.out_edges(t)
        for e in edges:
            if e.memlet is not None:
                spec.checks.append((e.memlet.container, e.memlet.subset, menv))

    def _contract_kernel(self, cp):
        """Implicit GEMM on DMMA (mma.sync.m16n8k4 f64): CTA tile 128 MF m x TN
        n, 8 warps of 16 MF m rows; K in BK-wide chunks staged in (dynamic) shared memory
        through affine gathers (address = row part + k part, both
        precomputed), double-buffered through registers.  The accumulators
        start from O's current value (the WCR add) and store once.  FP64
        tensor ops fuse multiply and add: within 1e-12 of the sequential
        reference sum, not bitwise."""
        spec = self.spec
        X, Y, O = cp["X"], cp["Y"], cp["O"]
        Mp, Kp, Np = cp["M"], cp["K"], cp["N"]
        ext, rng = cp["ext"], cp["rng"]
        decode = self._contract_decode(cp)

        Mtot = 1
        for q in Mp:
            Mtot *= ext[q]
        Ktot = 1
        for q in Kp:
            Ktot *= ext[q]
        Ntot = ext[Np]
        TN = 8 * min(4, -(-Ntot // 8))
        NF = TN // 8
        MF, BK = CONTRACT_MF, CONTRACT_BK  # m16 fragments per warp, k chunk
        ax, ay, ao = (self.arg(("ptr", X)), self.arg(("ptr", Y)), self.arg(("ptr", O)))
        for c in (X, Y, O):
            self.cont(c)
        cyn = cp["cy"][1].get(Np, 0)
        con = cp["co"][1].get(Np, 0)
        L = [f"// generated by paper_2107_00555_b200.codegen: contraction (DMMA implicit GEMM) "
             f"M={Mtot} N={Ntot} K={Ktot}",
             "struct B2Args { long long w[%d]; };" % max(1, len(spec.args)),
             "namespace {",
             "constexpr int MF = %d, TM = 128 * MF, BK = %d, TN = %d, NF = %d, APAD = 4, BPAD = 4;"
             % (MF, BK, TN, NF),
             f"constexpr long long MT = {Mtot}LL, NT = {Ntot}LL, KT = {Ktot}LL;",
             "__device__ __forceinline__ void b2c_dmma(double (&d)[4], double a0, double a1, "
             "double b0) {",
             '  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, '
             '{%4,%5}, {%6}, {%0,%1,%2,%3};\\n" : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) '
             ': "d"(a0), "d"(a1), "d"(b0));',
             "}",
             "__device__ __forceinline__ long long b2c_mx(unsigned m) { return "
             + decode(Mp, cp["cx"], "m") + "; }",
             "__device__ __forceinline__ long long b2c_kx(unsigned k) { return "
             + decode(Kp, cp["cx"], "k") + "; }",
             "__device__ __forceinline__ long long b2c_ky(unsigned k) { return "
             + decode(Kp, cp["cy"], "k") + "; }",
             "__device__ __forceinline__ long long b2c_mo(unsigned m) { return "
             + decode(Mp, cp["co"], "m") + "; }",
             "}  // namespace",
             f'extern "C" __global__ void __launch_bounds__(256) {spec.name}'
             f"(const __grid_constant__ B2Args a) {{",
             "  B2_PDL_ENTRY();",
             f"  const double *__restrict__ X = (const double *){ax} + {cp['cx'][0]}LL;",
             f"  const double *__restrict__ Y = (const double *){ay} + {cp['cy'][0]}LL;",
             f"  double *__restrict__ O = (double *){ao} + {cp['co'][0]}LL;",
             "  extern __shared__ __align__(16) double b2c_smem[];",
             "  double (*As)[TM][BK + APAD] = reinterpret_cast<double (*)[TM][BK + APAD]>(b2c_smem);",
             "  double (*Bs)[BK][TN + BPAD] = reinterpret_cast<double (*)[BK][TN + BPAD]>("
             "b2c_smem + 2 * TM * (BK + APAD));",
             "  long long *sMX = reinterpret_cast<long long *>("
             "b2c_smem + 2 * TM * (BK + APAD) + 2 * BK * (TN + BPAD));",
             "  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;",
             "  const int g = lane >> 2, t = lane & 3;",
             "  const long long ntiles = (NT + TN - 1) / TN;",
             "  for (long long tile = blockIdx.x; tile < ((MT + TM - 1) / TM) * ntiles; "
             "tile += gridDim.x) {",
             "    const long long m0 = (tile / ntiles) * TM, n0 = (tile % ntiles) * TN;",
             "    __syncthreads();",
             "    if (tid < TM) sMX[tid] = (m0 + tid < MT) ? b2c_mx((unsigned)(m0 + tid)) : 0LL;",
             "    __syncthreads();",
             # staging: A element e = tid + 256 r: row e / BK, col e % BK
             "    double ra[TM * BK / 256], rb[(BK * TN + 255) / 256];",
             "    auto load = [&](long long k0) {",
             "      // a thread stages one k column of A (8 rows) and one element of B",
             "      const int acol = tid % BK;",
             "      const long long ka = k0 + acol;",
             "      const long long kx = ka < KT ? b2c_kx((unsigned)ka) : 0LL;",
             "#pragma unroll",
             "      for (int r = 0; r < TM * BK / 256; ++r) {",
             "        const int row = tid / BK + (256 / BK) * r;",
             "        ra[r] = (m0 + row < MT && ka < KT) ? X[sMX[row] + kx] : 0.0;",
             "      }",
             "#pragma unroll",
             "      for (int r = 0; r < (BK * TN + 255) / 256; ++r) {",
             "        const int e = tid + 256 * r;",
             "        if (e < BK * TN) {",
             "          const int row = e / TN, col = e % TN;",
             "          const long long k = k0 + row, n = n0 + col;",
             f"          rb[r] = (k < KT && n < NT) ? Y[b2c_ky((unsigned)k) + {cyn}LL * "
             f"({rng[Np][0]}LL + {rng[Np][1]}LL * n)] : 0.0;",
             "        }",
             "      }",
             "    };",
             "    auto store = [&](int buf) {",
             "#pragma unroll",
             "      for (int r = 0; r < TM * BK / 256; ++r) {",
             "        As[buf][tid / BK + (256 / BK) * r][tid % BK] = ra[r];",
             "      }",
             "#pragma unroll",
             "      for (int r = 0; r < (BK * TN + 255) / 256; ++r) {",
             "        const int e = tid + 256 * r;",
             "        if (e < BK * TN) Bs[buf][e / TN][e % TN] = rb[r];",
             "      }",
             "    };",
             # accumulators start from O (the WCR add)
             "    double acc[MF][NF][4];",
             "    const int wm = warp * 16 * MF;",
             "#pragma unroll",
             "    for (int mf = 0; mf < MF; ++mf)",
             "#pragma unroll",
             "    for (int f = 0; f < NF; ++f)",
             "#pragma unroll",
             "      for (int h = 0; h < 2; ++h)",
             "#pragma unroll",
             "        for (int e2 = 0; e2 < 2; ++e2) {",
             "          const long long m = m0 + wm + 16 * mf + g + 8 * h, n = n0 + f * 8 + 2 * t + e2;",
             (f"          acc[mf][f][2 * h + e2] = 0.0; (void)m; (void)n;" if cp.get("init_zero") else
              f"          acc[mf][f][2 * h + e2] = (m < MT && n < NT) ? O[b2c_mo((unsigned)m) + {con}LL * "
              f"({rng[Np][0]}LL + {rng[Np][1]}LL * n)] : 0.0;"),
             "        }",
             "    load(0);",
             "    store(0);",
             "    __syncthreads();",
             "    const long long nk = (KT + BK - 1) / BK;",
             "    for (long long kc = 0; kc < nk; ++kc) {",
             "      const int cur = (int)(kc & 1);",
             "      if (kc + 1 < nk) load((kc + 1) * BK);",
             "#pragma unroll",
             "      for (int k4 = 0; k4 < BK; k4 += 4) {",
             "        double bf[NF];",
             "#pragma unroll",
             "        for (int f = 0; f < NF; ++f) bf[f] = Bs[cur][k4 + t][f * 8 + g];",
             "#pragma unroll",
             "        for (int mf = 0; mf < MF; ++mf) {",
             "          const double a0 = As[cur][wm + 16 * mf + g][k4 + t], "
             "a1 = As[cur][wm + 16 * mf + g + 8][k4 + t];",
             "#pragma unroll",
             "          for (int f = 0; f < NF; ++f) b2c_dmma(acc[mf][f], a0, a1, bf[f]);",
             "        }",
             "      }",
             "      if (kc + 1 < nk) store(cur ^ 1);",
             "      __syncthreads();",
             "    }",
             "#pragma unroll",
             "    for (int mf = 0; mf < MF; ++mf)",
             "#pragma unroll",
             "    for (int f = 0; f < NF; ++f)",
             "#pragma unroll",
             "      for (int h = 0; h < 2; ++h)",
             "#pragma unroll",
             "        for (int e2 = 0; e2 < 2; ++e2) {",
             "          const long long m = m0 + wm + 16 * mf + g + 8 * h, n = n0 + f * 8 + 2 * t + e2;",
             f"          if (m < MT && n < NT) O[b2c_mo((unsigned)m) + {con}LL * "
             f"({rng[Np][0]}LL + {rng[Np][1]}LL * n)] = acc[mf][f][2 * h + e2];",
             "        }",
             "  }",
             "}"]
        self._contract_checks(cp)
        spec.source = "\n".join(L) + "\n"
        spec.block = (256, 1, 1)
        spec.vec = 1
        spec.pdl = False
        spec.contract = {"M": Mtot, "N": Ntot, "K": Ktot, "TN": TN, "TM": 128 * MF}
        spec.smem = 8 * (2 * 128 * MF * (BK + 4) + 2 * BK * (TN + 4) + 128 * MF)
        return spec

    def _reduction_plan(self):
        """Reduction schedule for a parallel map whose only HBM writes are WCR
        commits (ir.py:72-91) that do not depend on some parameters R: each
        thread owns a point of the other parameters and runs R sequentially in
        a register accumulator (lexicographic order, bitwise equal to the
        reference when it owns the whole reduction), committing once."""
        grp = self.group
        if grp.schedule != "parallel" or not grp.params:
            return None
        if any(r is None for r in self.const_ranges):
            return None
        targets: dict = {}
        deps_all: set = set()
        reads: set = set()
        for mem in grp.members:
            for (c, w, wcr, depth, pt) in self.pl.member_accesses(mem, grp.params):
                if self.place(c) in ("reg", "private"):
                    continue  # thread-local: no cross-thread effect
                if not w:
                    reads.add(c)
                    continue
                if wcr is None or depth != 0 or pt is None or self.place(c) != "memory":
                    return None
                deps = {p for key in pt for (p, _) in key[1]}
                targets[(c, pt)] = (wcr, deps)
                deps_all |= deps
        if not targets or reads & {c for (c, _) in targets}:
            return None
        R = [p for p in grp.params if p not in deps_all]
        if not R:
            return None
        pout = [p for p in grp.params if p in deps_all]
        return R, pout, targets

    def _reduce_loop(self, R, pout, reg_decls, body) -> list:
        grp = self.group
        idx = {p: i for i, p in enumerate(grp.params)}
        nout = 1
        for p in pout:
            nout *= self.const_ranges[idx[p]][2]
        nred = 1
        for p in R:
            nred *= self.const_ranges[idx[p]][2]
        full = self.red_full
        C = 1 if full else max(1, min(-(-RED_THREADS // max(1, nout)), -(-nred // 16)))
        self.spec.red_threads = nout * C
        if full and RED_BLOCK and len(pout) >= 2:
            T = self.const_ranges[idx[pout[-1]]][2]
            if (2 <= T <= RED_BLOCK and nout // T >= 148 * 256
                    and all(t["exclusive"] for t in self.red.values())):
                return self._reduce_loop_blocked(R, pout, reg_decls, body, nout, T)
        if not full and nout <= 4096 and nout * nred <= (1 << 22) and SMALL_RED_CHUNK:
            # small latency-bound reductions (nbody's 100 x 100 pair forces,
            # a pow per term): short chunks, folded in-block, one launch
            C2 = min(-(-nred // SMALL_RED_CHUNK), 64)
            if C2 > C:
                self.spec.red_threads = nout * C2
                return self._reduce_loop_inblock(R, pout, reg_decls, body, nout, nred, C2)
        if not full and C <= 8:
            # few chunks per output: whole warps stay on one chunk of 32
            # consecutive outputs (coalesced / broadcast loads like the
            # thread-per-output layout) and the fold happens in-block
            return self._reduce_loop_inblock(R, pout, reg_decls, body, nout, nred, C)
        ob = self._red_out_block(pout, nout) if not full else 1
        if ob > 1:
            return self._reduce_loop_ob(R, pout, reg_decls, body, nout, nred, C, ob)
        L = [f"  constexpr b2_ll NOUT = {nout}LL, NRED = {nred}LL, NCH = {C}LL;",
             "  for (b2_ll f = (b2_ll)blockIdx.x * blockDim.x + threadIdx.x; f < NOUT * NCH; "
             "f += (b2_ll)gridDim.x * blockDim.x) {",
             "    b2_ll rem = f % NOUT;", "    const b2_ll ch = f / NOUT; (void)ch;"]
        for p in reversed(pout):
            i = idx[p]
            L.append(f"    const b2_ll q{i} = rem % rl{i}; rem /= rl{i};")
            L.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * q{i};")
        for t in self.red.values():
            a, ct = t["acc"], t["ct"]
            if full and t["exclusive"]:
                L.append(f"    {ct} {a} = {self._old(t)};")
            else:
                ident = {"add": "0", "mul": "1", "min": "b2_inf()", "max": "(-b2_inf())"}[t["wcr"]]
                if ct != "double" and t["wcr"] in ("min", "max"):
                    ident = "0"  # integer min/max: committed only when iterations ran
                L.append(f"    {ct} {a} = ({ct})({ident});")
        if full:
            for n, p in enumerate(R):
                i = idx[p]
                trip = self.const_ranges[i][2]
                L.append(f"    for (int j{i} = 0; j{i} < (int)rl{i}; ++j{i}) {{")
                L.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * j{i};")
        else:
            L.append("    const b2_ll lo = ch * NRED / NCH, hi = (ch + 1) * NRED / NCH;")
            # 32-bit induction variable when it fits: with a 64-bit one and
            # all-constexpr bounds, nvcc 12.9 (sm_100a) emitted a loop that never
            # terminated (reproduced standalone; int form is correct)
            it = "int" if nred < 2 ** 31 else "b2_ll"
            L.append(f"    for ({it} rf = ({it})lo; rf < ({it})hi; ++rf) {{")
            L.append("    b2_ll rr = rf;")
            for p in reversed(R):
                i = idx[p]
                if len(R) == 1:
                    L.append(f"    const b2_ll j{i} = rr;")  # lo..hi lies inside [0, rl)
                else:
                    L.append(f"    const b2_ll j{i} = rr % rl{i}; rr /= rl{i};")
                L.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * j{i};")
        L += reg_decls(4)
        L += body
        if full:
            for _ in R:
                L.append("    }")
        else:
            L.append("    }")
        self.spec.red_fin = []
        self.spec.red_nout, self.spec.red_nch = nout, C
        self.red_decode = [ln for ln in L if ln.strip().startswith(("const b2_ll q", "const b2_ll p_"))
                           and any(f"p_{p} " in ln or f"q{idx[p]} " in ln for p in pout)]
        for k, t in enumerate(self.red.values()):
            a = t["acc"]
            if full and t["exclusive"]:
                L.append(f"    {t['target']} = {a};")
            elif not full and t["ct"] == "double":
                # deterministic: chunk partials to a workspace, reduced in
                # chunk order by the companion _fin kernel (run-to-run
                # bitwise reproducible, like the reference, interp.py:153)
                ws = self.arg(("ptr", f"{self.spec.name}#ws{k}"))
                L.append(f"    ((double *){ws})[ch * NOUT + (f % NOUT)] = {a};")
                self.spec.red_fin.append((ws, t))
            else:
                cond = "" if full else "if (lo < hi) "
                L.append(f"    {cond}b2_atomic_{t['wcr']}(&{t['target']}, {a});")
        L.append("  }")
        return L

    def _red_out_block(self, pout, nout) -> int:
        """Outputs per thread for a chunked reduction whose every HBM read is
        the same for all outputs (azimint: radius[k], data[k] per bin): each
        loaded term then feeds RED_OUT_BLOCK accumulators (1: off)."""
        if RED_OUT_BLOCK < 2 or len(pout) != 1 or nout % RED_OUT_BLOCK:
            return 1
        if any(t["ct"] != "double" for t in self.red.values()):
            return 1
        grp = self.group
        for mem in grp.members:
            for (c, w, wcr, depth, pt) in self.pl.member_accesses(mem, grp.params):
                if w or self.place(c) != "memory":
                    continue
                if pt is None or any(p == pout[0] for key in pt for (p, _) in key[1]):
                    return 1
        return RED_OUT_BLOCK

    def _reduce_loop_ob(self, R, pout, reg_decls, body, nout, nred, C, OB) -> list:
        """The chunked reduction with OB consecutive outputs per thread: the
        body runs OB times per term with the output parameter stepped and
        its own accumulator (the loads are common subexpressions), partials
        to the workspace as usual (same per-output term order: bitwise equal
        to the one-output layout)."""
        grp = self.group
        idx = {p: i for i, p in enumerate(grp.params)}
        i0 = idx[pout[0]]
        names = [t["acc"] for t in self.red.values()]
        pat = re.compile(r"\b(" + "|".join(map(re.escape, names)) + r")\b")
        L = [f"  constexpr b2_ll NOUT = {nout}LL, NRED = {nred}LL, NCH = {C}LL;",
             f"  constexpr int OB = {OB};",
             "  constexpr b2_ll NOUTB = NOUT / OB;",
             "  for (b2_ll f = (b2_ll)blockIdx.x * blockDim.x + threadIdx.x; f < NOUTB * NCH; "
             "f += (b2_ll)gridDim.x * blockDim.x) {",
             "    const b2_ll qb = (f % NOUTB) * OB;", "    const b2_ll ch = f / NOUTB;"]
        for t in self.red.values():
            ident = {"add": "0", "mul": "1", "min": "b2_inf()", "max": "(-b2_inf())"}[t["wcr"]]
            L.append(f"    double {t['acc']}[OB];")
            L.append(f"#pragma unroll")
            L.append(f"    for (int ob_ = 0; ob_ < OB; ++ob_) {t['acc']}[ob_] = (double)({ident});")
        L.append("    const b2_ll lo = ch * NRED / NCH, hi = (ch + 1) * NRED / NCH;")
        it = "int" if nred < 2 ** 31 else "b2_ll"
        L.append(f"    for ({it} rf = ({it})lo; rf < ({it})hi; ++rf) {{")
        L.append("    b2_ll rr = rf;")
        for p in reversed(R):
            i = idx[p]
            if len(R) == 1:
                L.append(f"    const b2_ll j{i} = rr;")
            else:
                L.append(f"    const b2_ll j{i} = rr % rl{i}; rr /= rl{i};")
            L.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * j{i};")
        L.append("#pragma unroll")
        L.append("    for (int ob_ = 0; ob_ < OB; ++ob_) {")
        L.append(f"    const b2_ll q{i0} = qb + ob_;")
        L.append(f"    const b2_ll p_{pout[0]} = rb{i0} + rs{i0} * q{i0};")
        L += reg_decls(4)
        L += [pat.sub(lambda m: m.group(1) + "[ob_]", ln) for ln in body]
        L.append("    }")
        L.append("    }")
        self.spec.red_fin = []
        self.spec.red_nout, self.spec.red_nch = nout, C
        self.spec.red_threads = (nout // OB) * C
        self.red_decode = [f"    const b2_ll q{i0} = rem % rl{i0}; rem /= rl{i0};",
                           f"    const b2_ll p_{pout[0]} = rb{i0} + rs{i0} * q{i0};"]
        for k, t in enumerate(self.red.values()):
            ws = self.arg(("ptr", f"{self.spec.name}#ws{k}"))
            L.append("#pragma unroll")
            L.append(f"    for (int ob_ = 0; ob_ < OB; ++ob_) "
                     f"((double *){ws})[ch * NOUT + qb + ob_] = {t['acc']}[ob_];")
            self.spec.red_fin.append((ws, t))
        L.append("  }")
        return L

    def _march_prefetch(self, vec, by, ax) -> list:
        bx = self.spec.block[0]
        """L2 bulk prefetch (cp.async.bulk.prefetch.L2) of the rows of every
        read-only input the tile will touch, issued when the CTA picks the
        tile up: the march's demand loads then find most lines in L2, so far
        more bytes are in flight per SM than one load per thread allows."""
        grp = self.group
        out = []
        for c in sorted(self.read_set - self.written):
            if self.place(c) != "memory":
                continue
            shape = self.shapes[c]
            if len(shape) != 3:
                continue
            offs = []
            ok = True
            for mem in grp.members:
                for (cc, w, wcr, depth, pt) in self.pl.member_accesses(mem, grp.params):
                    if cc != c:
                        continue
                    if pt is None or len(pt) != 3:
                        ok = False
                        break
                    o = []
                    for d, (c0, co) in enumerate(pt):
                        if co != ((grp.params[d], 1),):
                            ok = False
                            break
                        o.append(c0)
                    if not ok:
                        break
                    offs.append(o)
                if not ok:
                    break
            if not ok or not offs:
                continue
            lo = [min(o[d] for o in offs) for d in range(3)]
            hi = [max(o[d] for o in offs) for d in range(3)]
            esz = 8 if self.g.containers[c].dtype in ("f64", "i64") else 4
            out += [
                "    {",
                f"      const b2_ll z0 = b2_max_ll(rb0 + tz * {vec} + ({lo[0]}LL), 0LL);",
                f"      const b2_ll z1 = b2_min_ll(rb0 + b2_min_ll(tz * {vec} + {vec - 1}, rl0 - 1) + ({hi[0]}LL), {shape[0] - 1}LL);",
                f"      const b2_ll y0 = b2_max_ll(rb1 + ty * {by} + ({lo[1]}LL), 0LL);",
                f"      const b2_ll y1 = b2_min_ll(rb1 + b2_min_ll(ty * {by} + {by - 1}, rl1 - 1) + ({hi[1]}LL), {shape[1] - 1}LL);",
                f"      const b2_ll x0 = b2_max_ll(rb2 + tx * {bx} - {ax} + ({lo[2]}LL), 0LL);",
                f"      const b2_ll x1 = b2_min_ll(rb2 + b2_min_ll(tx * {bx} - {ax} + {bx - 1}, rl2 - 1) + ({hi[2]}LL), {shape[2] - 1}LL);",
                "      const int ny = (int)(y1 - y0 + 1), nrow = (int)(z1 - z0 + 1) * ny;",
                f"      const b2_ll base = (b2_ll)(const char *)c_{c};",
                "      for (int r = threadIdx.y * blockDim.x + threadIdx.x; r < nrow; r += blockDim.x * blockDim.y) {",
                "        const int zz = r / ny, yy = r - zz * ny;",
                f"        const b2_ll row = (z0 + zz) * st_{c}_0 + (y0 + yy) * st_{c}_1;",
                f"        const b2_ll e0 = (row + x0) * {esz}LL, e1 = (row + x1 + 1) * {esz}LL;",
                "        const b2_ll a0 = (base + e0) & ~15LL, a1 = (base + e1 + 15) & ~15LL;",
                "        b2_prefetch_l2((const void *)a0, (unsigned)(a1 - a0));",
                "      }",
                "    }",
            ]
        return out

    def _reduce_loop_blocked(self, R, pout, reg_decls, body, nout, T) -> list:
        """Full reductions whose innermost output parameter is short (conv2d's
        output channel): each thread owns all T points of it, the reduction
        loops outside and the T points unrolled inside, so reads that do not
        depend on that parameter load once per T accumulations.  Per output
        the reduction still runs in lexicographic order (bitwise equal to the
        thread-per-output schedule)."""
        grp = self.group
        idx = {p: i for i, p in enumerate(grp.params)}
        pc = pout[-1]
        ic = idx[pc]
        self.spec.red_threads = nout // T
        accs = list(self.red.values())
        L = [f"  constexpr b2_ll NOUTB = {nout // T}LL;",
             "  for (b2_ll f = (b2_ll)blockIdx.x * blockDim.x + threadIdx.x; f < NOUTB; "
             "f += (b2_ll)gridDim.x * blockDim.x) {",
             "    b2_ll rem = f;"]
        for p in reversed(pout[:-1]):
            i = idx[p]
            L.append(f"    const b2_ll q{i} = rem % rl{i}; rem /= rl{i};")
            L.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * q{i};")
        for t in accs:
            L.append(f"    {t['ct']} {t['acc']}_v[{T}];")
        L.append("#pragma unroll")
        L.append(f"    for (int v = 0; v < {T}; ++v) {{")
        L.append(f"      const b2_ll p_{pc} = rb{ic} + rs{ic} * v;")
        for t in accs:
            L.append(f"      {t['acc']}_v[v] = {self._old(t)};")
        L.append("    }")
        for n, p in enumerate(R):
            i = idx[p]
            L.append(f"    for (int j{i} = 0; j{i} < (int)rl{i}; ++j{i}) {{")
            L.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * j{i};")
        L.append("#pragma unroll")
        L.append(f"    for (int v = 0; v < {T}; ++v) {{")
        L.append(f"    const b2_ll p_{pc} = rb{ic} + rs{ic} * v;")
        for t in accs:
            L.append(f"    {t['ct']} {t['acc']} = {t['acc']}_v[v];")
        L += reg_decls(4)
        L += body
        for t in accs:
            L.append(f"    {t['acc']}_v[v] = {t['acc']};")
        L.append("    }")
        for _ in R:
            L.append("    }")
        L.append("#pragma unroll")
        L.append(f"    for (int v = 0; v < {T}; ++v) {{")
        L.append(f"      const b2_ll p_{pc} = rb{ic} + rs{ic} * v;")
        for t in accs:
            L.append(f"      {t['target']} = {t['acc']}_v[v];")
        L.append("    }")
        L.append("  }")
        self.spec.red_fin = []
        self.spec.red_nout, self.spec.red_nch = nout, 1
        self.red_decode = []
        return L

    def _reduce_loop_inblock(self, R, pout, reg_decls, body, nout, nred, C) -> list:
        """Chunked reduction with every output's C chunks in one CTA: chunk
        partials meet in shared memory and the chunk-0 thread folds them in
        chunk order (deterministic, one kernel — no workspace pass)."""
        grp = self.group
        idx = {p: i for i, p in enumerate(grp.params)}
        opb = 256 // C
        self.spec.red_threads = -(-nout // opb) * 256
        dts = [t for t in self.red.values() if t["ct"] == "double"]
        L = [f"  constexpr b2_ll NOUT = {nout}LL, NRED = {nred}LL;",
             f"  constexpr int NCH = {C}, OPB = {opb};",
             f"  __shared__ double red_sm[{max(1, len(dts))}][256];",
             "  for (b2_ll ob = blockIdx.x; ob * OPB < NOUT; ob += gridDim.x) {",
             "    const int ol = (int)threadIdx.x % OPB, ch = (int)threadIdx.x / OPB;",
             "    const b2_ll fo = ob * OPB + ol;",
             "    const bool valid = (int)threadIdx.x < OPB * NCH && fo < NOUT;",
             "    b2_ll rem = valid ? fo : 0;"]
        for p in reversed(pout):
            i = idx[p]
            L.append(f"    const b2_ll q{i} = rem % rl{i}; rem /= rl{i};")
            L.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * q{i};")
        for t in self.red.values():
            ident = {"add": "0", "mul": "1", "min": "b2_inf()", "max": "(-b2_inf())"}[t["wcr"]]
            if t["ct"] != "double" and t["wcr"] in ("min", "max"):
                ident = "0"  # integer min/max: committed only when iterations ran
            L.append(f"    {t['ct']} {t['acc']} = ({t['ct']})({ident});")
        L.append("    const b2_ll lo = valid ? (b2_ll)ch * NRED / NCH : 0;")
        L.append("    const b2_ll hi = valid ? ((b2_ll)ch + 1) * NRED / NCH : 0;")
        it = "int" if nred < 2 ** 31 else "b2_ll"
        L.append(f"    for ({it} rf = ({it})lo; rf < ({it})hi; ++rf) {{")
        L.append("    b2_ll rr = rf;")
        for p in reversed(R):
            i = idx[p]
            if len(R) == 1:
                L.append(f"    const b2_ll j{i} = rr;")
            else:
                L.append(f"    const b2_ll j{i} = rr % rl{i}; rr /= rl{i};")
            L.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * j{i};")
        L += reg_decls(4)
        L += body
        L.append("    }")
        for k, t in enumerate(dts):
            L.append(f"    red_sm[{k}][threadIdx.x] = {t['acc']};")
        for t in self.red.values():
            if t["ct"] != "double":  # integer WCR: associative, atomics stay exact
                L.append(f"    if (lo < hi) b2_atomic_{t['wcr']}(&{t['target']}, {t['acc']});")
        L.append("    __syncthreads();")
        L.append("    if (valid && ch == 0) {")
        for k, t in enumerate(dts):
            op = t["wcr"]
            L.append(f"      double s{k} = red_sm[{k}][ol];")
            L.append(f"      for (int c = 1; c < NCH; ++c) s{k} = b2_op_{op}(s{k}, "
                     f"red_sm[{k}][c * OPB + ol]);")
            if t["exclusive"]:
                L.append(f"      {t['target']} = b2_op_{op}({self._old(t)}, s{k});")
            else:
                L.append(f"      b2_atomic_{op}(&{t['target']}, s{k});")
        L.append("    }")
        L.append("    __syncthreads();")
        L.append("  }")
        self.spec.red_fin = []
        return L

    def _reduce_fin(self, pro) -> list:
        """Companion kernel of a chunked reduction: per output, the chunk
        partials folded in a fixed order into the target with its WCR.  Many
        chunks: one CTA per output, 256 contiguous chunk ranges then thread 0
        over the 256 sums; few chunks: one thread per output."""
        spec = self.spec
        ident = {"add": "0.0", "mul": "1.0", "min": "b2_inf()", "max": "(-b2_inf())"}
        per_block = spec.red_nch >= 64
        spec.red_fin_block = per_block
        L = [f'extern "C" __global__ void __launch_bounds__(256) '
             f"{spec.name}_fin(const __grid_constant__ B2Args a) {{", "  B2_PDL_ENTRY();"]
        L += [ln for ln in pro[2:] if "pv_" not in ln and "tflat" not in ln]
        L.append(f"  constexpr b2_ll NOUT = {spec.red_nout}LL;")
        L.append(f"  constexpr int NCH = {spec.red_nch};")
        if per_block:
            L += ["  __shared__ double red[256];",
                  "  constexpr int PER = (NCH + 255) / 256;",
                  "  for (b2_ll f = blockIdx.x; f < NOUT; f += gridDim.x) {",
                  "    b2_ll rem = f; (void)rem;"]
        else:
            L += ["  for (b2_ll f = (b2_ll)blockIdx.x * blockDim.x + threadIdx.x; f < NOUT; "
                  "f += (b2_ll)gridDim.x * blockDim.x) {",
                  "    b2_ll rem = f; (void)rem;"]
        L += self.red_decode
        for ws, t in spec.red_fin:
            w = f"((const double *){ws})"
            op, acc = t["wcr"], f"s_{t['acc']}"
            if per_block:
                L += [f"    double {acc} = {ident[op]};",
                      "    {",
                      "      const int c0 = (int)threadIdx.x * PER;",
                      "      const int c1 = c0 + PER < NCH ? c0 + PER : NCH;",
                      f"      for (int c = c0; c < c1; ++c) {acc} = b2_op_{op}({acc}, {w}[c * NOUT + f]);",
                      "    }",
                      f"    red[threadIdx.x] = {acc};",
                      "    __syncthreads();",
                      "    if (threadIdx.x == 0) {",
                      f"      double t = red[0];",
                      f"      for (int i = 1; i < 256; ++i) t = b2_op_{op}(t, red[i]);",
                      f"      {t['target']} = b2_op_{op}({self._old(t)}, t);",
                      "    }",
                      "    __syncthreads();"]
            else:
                L += [f"    double {acc} = {w}[f];",
                      f"    for (int c = 1; c < NCH; ++c) {acc} = b2_op_{op}({acc}, {w}[c * NOUT + f]);",
                      f"    {t['target']} = b2_op_{op}({self._old(t)}, {acc});"]
        L += ["  }", "}"]
        return L

    def _rowred_plan(self):
        """Row-reduction schedule for a parallel map whose WCR targets do not
        depend on its last (contiguous) parameter L but whose other memory
        writes are full points (softmax: ``ex = exp(x - mx)`` plus
        ``sm += ex`` over L).  One warp per output row: lanes stride L
        (coalesced loads/stores), accumulate in registers, combine with a
        fixed xor-shuffle tree and commit once.  The sum is re-associated
        (within the rel_err 1e-12 contract)."""
        grp = self.group
        k = len(grp.params)
        if grp.schedule != "parallel" or k < 2 or any(r is None for r in self.const_ranges):
            return None
        if self.const_ranges[-1][2] < 32:
            return None
        last = grp.params[-1]
        targets: dict = {}
        reads: dict = {}
        pointw: dict = {}
        for mem in grp.members:
            for (c, w, wcr, depth, pt) in self.pl.member_accesses(mem, grp.params):
                if not w:
                    reads.setdefault(c, set()).add(pt)
                    continue
                if self.place(c) == "reg":
                    continue
                if depth != 0 or pt is None or self.place(c) != "memory":
                    return None
                deps = {p for key in pt for (p, _) in key[1]}
                if wcr is None:
                    if deps != set(grp.params) or pointw.get(c, pt) != pt:
                        return None
                    pointw[c] = pt
                    continue
                if last in deps or self.g.containers[c].dtype != "f64":
                    return None
                targets[(c, pt)] = (wcr, deps)
        if not targets:
            return None
        if set(reads) & {c for (c, _) in targets}:
            return None
        for c, pt in pointw.items():  # a written container is only re-read at its own point
            if reads.get(c, {pt}) != {pt}:
                return None
        self.rowred_pointw = dict(pointw)
        return [last], list(grp.params[:-1]), targets

    def _last_param_contiguous(self) -> bool:
        """Some HBM read walks the map's last parameter along its contiguous
        dimension with unit stride, and no read has it in another dimension."""
        grp = self.group
        last = grp.params[-1]
        found = False
        for mem in grp.members:
            for (c, w, wcr, depth, pt) in self.pl.member_accesses(mem, grp.params):
                if w or self.place(c) != "memory":
                    continue
                if pt is None:
                    return False
                for d, key in enumerate(pt):
                    co = dict(key[1])
                    if last in co:
                        if d != len(pt) - 1 or co[last] != 1:
                            return False
                        found = True
        return found

    def _epilogue_plan(self, B):
        """Map group ``B`` (the next op) runs as the epilogue of this row
        reduction when it iterates the same space, reads this group's
        point-written transients T only at their point and the reduction
        targets R only at the row's point, writes full points of containers
        this group does not touch, and no other op reads T: each warp keeps
        its row of T in registers (T never reaches HBM) and evaluates B from
        them and the reduced R (softmax: ex / sm).  Same tasklets, same
        values: bitwise equal to the two launches."""
        A = self.group
        if (not isinstance(B, P.MapGroup) or B.schedule != "parallel"
                or len(B.params) != len(A.params) or B.idx in self.pl.in_region):
            return None
        rb = [_const_range(self.pl, r) for r in B.ranges]
        if rb != self.const_ranges:
            return None
        TV = -(-self.const_ranges[-1][2] // 32)
        if TV > 32:
            return None
        ren = dict(zip(B.params, A.params))

        def rn(pt):
            return tuple((c0, tuple((ren.get(p, p), k) for p, k in co)) for c0, co in pt)

        Ts = {c: pt for c, pt in self.rowred_pointw.items() if self.g.containers[c].transient
              and self.g.containers[c].lifetime != "persistent"}
        if not Ts or set(Ts) != set(self.rowred_pointw):
            return None
        R = {c: pt for (c, pt) in self.red_targets}
        # every reduction target must be exclusive to its row (one warp
        # commits it), so the warp holds the final value
        if any(deps != set(self.red_pout) for (_, deps) in self.red_targets.values()):
            return None
        written_A = set(Ts) | set(R)
        touched_A = set()
        for mem in A.members:
            for (c, w, wcr, depth, pt) in self.pl.member_accesses(mem, A.params):
                touched_A.add(c)
        for mem in B.members:
            for (c, w, wcr, depth, pt) in self.pl.member_accesses(mem, B.params):
                if depth != 0 or pt is None:
                    return None
                if not w:
                    if c in Ts:
                        if rn(pt) != Ts[c]:
                            return None
                    elif c in R:
                        if rn(pt) != R[c]:
                            return None
                    elif c in written_A:
                        return None
                    continue
                if wcr is not None or c in touched_A:
                    return None
                deps = {p for key in pt for (p, _) in key[1]}
                if deps != set(B.params):
                    return None
        for op in self.pl.all_ops:
            if op.idx in (A.idx, B.idx):
                continue
            if set(self.pl.op_reads.get(op.idx, set())) & set(Ts):
                return None
        return {"B": B, "T": sorted(Ts), "TV": TV}

    def _rowred_prefetch(self, pout) -> list:
        """Lane 0 of each warp issues one L2 bulk prefetch per read-only
        input row the warp's next row will stream (softmax: x[i, j, k, :],
        4 KB), so the next row's demand loads find their lines in L2 while
        this row's exp / shuffle / epilogue run.  Only inputs read at one
        point, whose last dimension follows the row parameter with unit
        coefficient and whose other dimensions follow row-output parameters
        (or constants); a hint only, results unchanged."""
        grp = self.group
        idx = {p: i for i, p in enumerate(grp.params)}
        last = grp.params[-1]
        iL = idx[last]
        out = []
        for c in sorted(self.read_set - self.written):
            if self.place(c) != "memory":
                continue
            pts = set()
            for mem in grp.members:
                for (cc, w, wcr, depth, pt) in self.pl.member_accesses(mem, grp.params):
                    if cc == c:
                        pts.add(pt)
            if len(pts) != 1 or None in pts:
                continue
            pt = next(iter(pts))
            nd = len(pt)
            if nd < 1 or pt[-1][1] != ((last, 1),):
                continue
            terms, ok = [], True
            for d, (c0, co) in enumerate(pt[:-1]):
                if co == ():
                    terms.append(f"({c0}LL) * st_{c}_{d}")
                elif len(co) == 1 and co[0][1] == 1 and co[0][0] in pout:
                    terms.append(f"(pn_{co[0][0]} + ({c0}LL)) * st_{c}_{d}")
                else:
                    ok = False
                    break
            if not ok:
                continue
            c0L = pt[-1][0]
            esz = 8 if self.g.containers[c].dtype in ("f64", "i64") else 4
            terms.append(f"(rb{iL} + ({c0L}LL)) * st_{c}_{nd - 1}")
            out.append(f"      {{ const b2_ll e0 = {' + '.join(terms)};")
            out.append(f"        const b2_ll e1 = e0 + (rl{iL} - 1) * rs{iL} * st_{c}_{nd - 1} + 1;")
            out.append(f"        const b2_ll a0 = ((b2_ll)(const char *)c_{c} + e0 * {esz}LL) & ~15LL;")
            out.append(f"        const b2_ll a1 = ((b2_ll)(const char *)c_{c} + e1 * {esz}LL + 15) & ~15LL;")
            out.append("        if (a1 > a0 && a1 - a0 <= 65536) b2_prefetch_l2((const void *)a0, (unsigned)(a1 - a0)); }")
        if not out:
            return []
        L = ["    if (lane == 0) {",
             "      const b2_ll rown = row + (((b2_ll)gridDim.x * blockDim.x) >> 5);",
             "      if (rown < NOUT) {",
             "      b2_ll remn = rown;"]
        for p in reversed(pout):
            i = idx[p]
            L.append(f"      const b2_ll qn{i} = remn % rl{i}; remn /= rl{i};")
            L.append(f"      const b2_ll pn_{p} = rb{i} + rs{i} * qn{i};")
        for p in pout:
            L.append(f"      (void)pn_{p};")
        return L + out + ["      }", "    }"]

    def _rowred_loop(self, pout, reg_decls, body) -> list:
        grp = self.group
        idx = {p: i for i, p in enumerate(grp.params)}
        nout = 1
        for p in pout:
            nout *= self.const_ranges[idx[p]][2]
        self.spec.red_threads = nout * 32
        iL = len(grp.params) - 1
        L = [f"  constexpr b2_ll NOUT = {nout}LL;",
             "  const int lane = threadIdx.x & 31;",
             "  for (b2_ll row = ((b2_ll)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < NOUT;",
             "       row += ((b2_ll)gridDim.x * blockDim.x) >> 5) {",
             "    b2_ll rem = row;"]
        for p in reversed(pout):
            i = idx[p]
            L.append(f"    const b2_ll q{i} = rem % rl{i}; rem /= rl{i};")
            L.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * q{i};")
        if ROWRED_PF:
            L += self._rowred_prefetch(pout)
        for t in self.red.values():
            ident = {"add": "0", "mul": "1", "min": "b2_inf()", "max": "(-b2_inf())"}[t["wcr"]]
            L.append(f"    {t['ct']} {t['acc']} = ({t['ct']})({ident});")
        pL = grp.params[-1]
        if self.epi is not None:
            TV = self.epi["TV"]
            for T in self.epi["T"]:
                L.append(f"    {CT[self.g.containers[T].dtype]} tb_{T}[{TV}];")
            L.append("#pragma unroll")
            L.append(f"    for (int v = 0; v < {TV}; ++v) {{")
            L.append(f"    const int j{iL} = lane + 32 * v;")
            L.append(f"    if (j{iL} >= (int)rl{iL}) break;")
        elif self.hoisted:
            T = self.const_ranges[-1][2] // 32
            for name, ct, expr in self.hoisted:
                L.append(f"    {ct} {name}[{T}];")
            L.append("#pragma unroll")
            L.append(f"    for (int v = 0; v < {T}; ++v) {{")
            L.append(f"    const int j{iL} = lane + 32 * v;")
            L.append(f"    const b2_ll p_{pL} = rb{iL} + rs{iL} * j{iL};")
            for name, _, expr in self.hoisted:
                L.append(f"    {name}[v] = {expr};")
            L.append("    }")
            L.append("#pragma unroll")
            L.append(f"    for (int v = 0; v < {T}; ++v) {{")
            L.append(f"    const int j{iL} = lane + 32 * v;")
        else:
            if ROWRED_UNROLL > 1:
                L.append(f"#pragma unroll {ROWRED_UNROLL}")
            L.append(f"    for (int j{iL} = lane; j{iL} < (int)rl{iL}; j{iL} += 32) {{")
        L.append(f"    const b2_ll p_{pL} = rb{iL} + rs{iL} * j{iL};")
        L += reg_decls(4)
        L += body
        L.append("    }")
        for t in self.red.values():
            a = t["acc"]
            L.append(f"    for (int o = 16; o > 0; o >>= 1) {a} = b2_op_{t['wcr']}({a}, "
                     f"__shfl_xor_sync(0xffffffffu, {a}, o));")
        if self.epi is not None:
            # the xor tree left every lane with the reduced value: every lane
            # forms the committed value (old (+) acc, exclusive targets only),
            # lane 0 stores it, the epilogue reads it from the register
            for t in self.red.values():
                L.append(f"    {t['acc']} = b2_op_{t['wcr']}({self._old(t)}, {t['acc']});")
            L.append("    if (lane == 0) {")
            for t in self.red.values():
                L.append(f"      {t['target']} = {t['acc']};")
            L.append("    }")
        else:
            L.append("    if (lane == 0) {")
            for t in self.red.values():
                if t["exclusive"]:
                    L.append(f"      {t['target']} = b2_op_{t['wcr']}({self._old(t)}, {t['acc']});")
                else:
                    L.append(f"      b2_atomic_{t['wcr']}(&{t['target']}, {t['acc']});")
            L.append("    }")
        if self.epi is not None:
            L.append("#pragma unroll")
            L.append(f"    for (int v = 0; v < {self.epi['TV']}; ++v) {{")
            L.append(f"    const int j{iL} = lane + 32 * v;")
            L.append(f"    if (j{iL} >= (int)rl{iL}) break;")
            L.append(f"    const b2_ll p_{pL} = rb{iL} + rs{iL} * j{iL};")
            L += reg_decls(4)
            L += [ln[2:] if ln.startswith("  ") else ln for ln in self.epi_body]
            L.append("    }")
        L.append("  }")
        return L

    def _tma3_loop(self, reg_decls, body: list) -> list:
        """tma3 mode (3-D sweeps whose read-only inputs are read at constant
        offsets within +-1): each CTA of a persistent, balanced grid owns a
        contiguous run of (tile, plane) units — tiles of T3_TK x T3_TJ
        points over dims (1, 2), planes along dim 0 — and marches it.

        Warp-specialised pipeline: one producer warp streams every plane of
        every staged input into shared memory ONCE, as one
        cp.async.bulk.tensor.3d box (tile + halo, zero-filled outside the
        container), into a ring of T3_S slots; ``full[s]`` (expect_tx = the
        boxes' bytes) tells the consumer warps a slot has landed, ``empty[s]``
        (one arrival per consumer warp) tells the producer it may be
        refilled.  Consumer warps compute their rows of each plane from the
        window of span+1 slots (the tasklet chain unchanged, same op order as
        every other mode: bitwise equal) and store straight to HBM; no
        CTA-wide barrier in the steady state."""
        grp = self.group
        spec = self.spec
        L: list[str] = []
        st0 = next(iter(self.stencil.values()))
        mins, maxs = st0["min"], st0["max"]
        span = maxs[0] - mins[0]
        halo_j = maxs[1] - mins[1]
        halo_k = maxs[2] - mins[2]
        rl1, rl2 = self.const_ranges[1][2], self.const_ranges[2][2]
        ntx = -(-rl2 // 64)
        tk = -(-rl2 // ntx)
        # box rows start on 32-byte DRAM sectors (tile width a multiple of 4)
        # and are a 16-byte multiple long (TMA)
        tk = -(-tk // 4) * 4
        if (tk + halo_k) % 2:
            tk += 1
        tk = min(tk, 64)
        ntx = -(-rl2 // tk)
        cw = spec.block[1] - 1  # consumer warps (the last warp produces)
        tj = max(cw, min(TMA3_TJ // cw * cw, -(-rl1 // cw) * cw))
        sk, sj = tk + halo_k, tj + halo_j
        slot = -(-(sk * sj * 8) // 128) * 128 // 8  # doubles per slot, 128-B aligned
        S = span + 1 + TMA3_PREF
        conts = list(self.stencil)
        spec.tmaps = [(c, (sk, sj, 1)) for c in conts]
        spec.smem = len(conts) * S * slot * 8
        nty = -(-rl1 // tj)
        rl0 = self.const_ranges[0][2]
        units = ntx * nty * rl0
        if TMA3_CHUNK:
            # one CTA per (tile, run of planes), tiles fastest: the hardware
            # scheduler balances the SMs and a chunk's first (halo) planes
            # were read by the previous wave moments ago (L2 hits)
            nch = -(-rl0 // TMA3_CHUNK)
            chunk = -(-rl0 // nch)
            spec.grid_cap = ntx * nty * nch
        else:
            chunk = 0
            spec.grid_cap = max(1, min(units, 148 * TMA3_CTAS))
        box_bytes = sk * sj * 8 * len(conts)
        L.append(f"  constexpr int T3_S = {S}, T3_SK = {sk}, T3_SLOT = {slot}, T3_TK = {tk}, "
                 f"T3_CW = {cw};")
        L.append(f"  constexpr b2_ll T3_NTX = {ntx}, T3_NT = {ntx * nty};")
        L.append(f"  constexpr b2_ll T3_W = T3_NT * rl0;")
        L.append("  extern __shared__ __align__(1024) double t3_smem[];")
        L.append("  __shared__ __align__(8) unsigned long long t3_full[T3_S], t3_empty[T3_S];")
        for i, c in enumerate(conts):
            L.append(f"  const double *tsm_{c} = t3_smem + {i} * T3_S * T3_SLOT;")
        L.append("  if (threadIdx.y == 0 && threadIdx.x == 0) {")
        L.append("    for (int q = 0; q < T3_S; ++q) {")
        L.append("      b2_mbar_init(&t3_full[q], 1);")
        L.append("      b2_mbar_init(&t3_empty[q], T3_CW);")
        L.append("    }")
        L.append("  }")
        L.append("  __syncthreads();")
        if chunk:
            L.append("  const b2_ll t3_tile = blockIdx.x % T3_NT, t3_ch = blockIdx.x / T3_NT;")
            L.append(f"  const b2_ll u0 = t3_tile * rl0 + t3_ch * {chunk};")
            L.append(f"  const b2_ll uend = t3_tile * rl0 + ((t3_ch + 1) * {chunk} < rl0 ? "
                     f"(t3_ch + 1) * {chunk} : rl0);")
        else:
            L.append("  const b2_ll u0 = (b2_ll)blockIdx.x * T3_W / gridDim.x;")
            L.append("  const b2_ll uend = ((b2_ll)blockIdx.x + 1) * T3_W / gridDim.x;")
        # ---- producer warp
        L.append("  if (threadIdx.y == T3_CW) {")
        L.append("    if (threadIdx.x == 0) {")
        for i in range(len(conts)):
            L.append(f'      asm volatile("prefetch.tensormap [%0];" ::"l"((unsigned long long)&a.tm[{i}]) : "memory");')
        L.append("      unsigned t = 0;")
        L.append("      for (b2_ll u = u0; u < uend;) {")
        L.append("        const b2_ll tile = u / rl0, i_start = u % rl0;")
        L.append("        const b2_ll n_it = ((rl0 < i_start + (uend - u)) ? rl0 : i_start + (uend - u)) - i_start;")
        L.append(f"        const b2_ll kx0 = (tile % T3_NTX) * T3_TK, jy0 = (tile / T3_NTX) * {tj};")
        L.append(f"        const int g0 = (int)(rb0 + i_start + ({mins[0]})), gj = (int)(rb1 + jy0 + ({mins[1]})), "
                 f"gk = (int)(rb2 + kx0 + ({mins[2]}));")
        if TMA3_L2PF:
            # L2 prefetch of the planes ahead of the ring (no shared memory:
            # the ring's loads then hit L2)
            L.append(f"        for (int q = 0; q < {TMA3_L2PF} && q < n_it + {span}; ++q) {{")
            for i in range(len(conts)):
                L.append("          asm volatile(\"cp.async.bulk.prefetch.tensor.3d.L2.global.tile "
                         f"[%0, {{%1, %2, %3}}];\" :: \"l\"((unsigned long long)&a.tm[{i}]), "
                         "\"r\"(gk), \"r\"(gj), \"r\"(g0 + q) : \"memory\");")
            L.append("        }")
        L.append(f"        for (int q = 0; q < n_it + {span}; ++q, ++t) {{")
        L.append("          const unsigned s = t % T3_S;")
        if TMA3_L2PF:
            L.append(f"          if (q + {TMA3_L2PF} < n_it + {span}) {{")
            for i in range(len(conts)):
                L.append("            asm volatile(\"cp.async.bulk.prefetch.tensor.3d.L2.global.tile "
                         f"[%0, {{%1, %2, %3}}];\" :: \"l\"((unsigned long long)&a.tm[{i}]), "
                         f"\"r\"(gk), \"r\"(gj), \"r\"(g0 + q + {TMA3_L2PF}) : \"memory\");")
            L.append("          }")
        L.append("          b2_mbar_wait(&t3_empty[s], ((t / T3_S) & 1u) ^ 1u);")
        L.append("          const unsigned fb = (unsigned)__cvta_generic_to_shared(&t3_full[s]);")
        L.append(f'          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), '
                 f'"r"({box_bytes}u) : "memory");')
        for i, c in enumerate(conts):
            L.append("          asm volatile(\"cp.async.bulk.tensor.3d.shared::cluster.global.tile."
                     "mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\" "
                     f":: \"r\"((unsigned)__cvta_generic_to_shared(tsm_{c} + s * T3_SLOT)), "
                     f"\"l\"((unsigned long long)&a.tm[{i}]), \"r\"(gk), \"r\"(gj), "
                     "\"r\"(g0 + q), \"r\"(fb) : \"memory\");")
        L.append("        }")
        L.append("        u += n_it;")
        L.append("      }")
        L.append("    }")
        L.append("  } else {")
        # ---- consumer warps
        L.append("    unsigned t = 0;")
        L.append("    for (b2_ll u = u0; u < uend;) {")
        L.append("      const b2_ll tile = u / rl0, i_start = u % rl0;")
        L.append("      const b2_ll n_it = ((rl0 < i_start + (uend - u)) ? rl0 : i_start + (uend - u)) - i_start;")
        L.append(f"      const b2_ll kx0 = (tile % T3_NTX) * T3_TK, jy0 = (tile / T3_NTX) * {tj};")
        L.append("      for (b2_ll it = 0; it < n_it; ++it) {")
        L.append(f"        for (unsigned w = (it == 0 ? t : t + {span}); w <= t + {span}; ++w)")
        L.append("          b2_mbar_wait(&t3_full[w % T3_S], (w / T3_S) & 1u);")
        for o in range(span + 1):
            L.append(f"        const int sl_{o} = (int)((t + {o}) % T3_S) * T3_SLOT;")
        L.append(f"        const b2_ll p_{grp.params[0]} = rb0 + i_start + it;")
        L.append("#pragma unroll")
        L.append(f"        for (int r = 0; r < {tj // cw}; ++r) {{")
        L.append(f"        const int ly = threadIdx.y + {cw} * r;")
        L.append(f"        if (jy0 + ly >= {rl1}LL) break;")
        L.append(f"        const b2_ll p_{grp.params[1]} = rb1 + jy0 + ly;")
        L.append("#pragma unroll")
        L.append("        for (int v = 0; v < 2; ++v) {")
        L.append("          const int lx = threadIdx.x + 32 * v;")
        L.append(f"          if (lx >= T3_TK || kx0 + lx >= {rl2}LL) break;")
        L.append(f"          const b2_ll p_{grp.params[2]} = rb2 + kx0 + lx;")
        L += reg_decls(10)
        L += ["        " + ln for ln in body]
        L.append("        }")
        L.append("        }")
        # release the oldest slot of the window (and at the end of the run
        # of planes, the span slots above it too)
        L.append("        __syncwarp();")
        L.append(f"        const unsigned rel = (it + 1 == n_it) ? {span} + 1u : 1u;")
        L.append("        if (threadIdx.x == 0)")
        L.append("          for (unsigned q = 0; q < rel; ++q)")
        L.append("            asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" ::\"r\"("
                 "(unsigned)__cvta_generic_to_shared(&t3_empty[(t + q) % T3_S])) : \"memory\");")
        L.append("        t += rel;")
        L.append("      }")
        L.append("      u += n_it;")
        L.append("    }")
        L.append("  }")
        return L

    def _stencil_offsets(self, m: sdfg.Memlet, env: dict) -> tuple:
        offs = []
        for d, (b, _, _) in enumerate(m.subset):
            a = symexpr.affine(b, tuple(env), self.pl.fixed)
            offs.append(a[0])
        return tuple(offs)

    def _stencil_analysis(self) -> dict:
        """Containers read (never written) by the group only at constant
        offsets from the point, dimension d indexed by parameter d: these are
        staged through a shared-memory plane ring (stencil mode)."""
        grp = self.group
        k = len(grp.params)
        reads: dict[str, set] = {}
        written = set()
        for mem in grp.members:
            for (c, w, wcr, depth, pt) in self.pl.member_accesses(mem, grp.params):
                if w:
                    written.add(c)
                    continue
                if depth != 0 or pt is None:
                    reads[c] = None
                    continue
                if reads.get(c, set()) is None:
                    continue
                offs = []
                ok = len(pt) == k
                for d, key in enumerate(pt if ok else ()):
                    c0, co = key
                    if co != ((grp.params[d], 1),):
                        ok = False
                        break
                    offs.append(c0)
                if not ok:
                    reads[c] = None
                else:
                    reads.setdefault(c, set()).add(tuple(offs))
        out = {}
        for c, offs in reads.items():
            if offs is None or c in written or self.place(c) != "memory":
                continue
            if len(self.shapes[c]) != k:
                continue
            lo = tuple(min(o[d] for o in offs) for d in range(k))
            hi = tuple(max(o[d] for o in offs) for d in range(k))
            if lo == hi:
                continue  # no halo: plain loads are as good
            if max(h - l for h, l in zip(hi, lo)) > 4:
                continue
            out[c] = {"offs": offs, "min": lo, "max": hi}
        if out:  # one plane ring geometry shared by every staged container
            mins = tuple(min(st["min"][d] for st in out.values()) for d in range(k))
            maxs = tuple(max(st["max"][d] for st in out.values()) for d in range(k))
            for st in out.values():
                st["min"], st["max"] = mins, maxs
        return out

    # -- helpers ---------------------------------------------------------------

    def emit(self, s: str):
        self.lines.append(" " * self.ind + s)

    def fresh(self, base: str) -> str:
        self.uid += 1
        return f"{base}_{self.uid}"

    def arg(self, desc) -> str:
        i = self.spec.arg_index(desc)
        return f"a.w[{self.arg_base + i}]"

    def sym(self, name: str) -> str:
        if name not in self.spec.syms:
            self.spec.syms.append(name)
        return f"s_{name}"

    def name_of(self, env):
        def f(n):
            if n in env:
                return env[n]
            if n in self.g.containers:
                raise P.PlanError(f"container '{n}' used as an index symbol")
            return self.sym(n)
        return f

    def cont(self, name: str):
        if name not in self.spec.containers:
            self.spec.containers.append(name)
        return self.g.containers[name]

    def place(self, name: str) -> str:
        if name in self.place_override:
            return self.place_override[name]
        return self.pl.placement.get(name, "memory")

    def offset(self, name: str, idx_codes: list[str]) -> str:
        c = self.cont(name)
        if not idx_codes:
            return "0LL"
        terms = []
        for d, ic in enumerate(idx_codes):
            terms.append(f"({ic}) * st_{name}_{d}")
        return " + ".join(terms)

    def ptr(self, name: str) -> str:
        if name in self.ptr_override:
            return self.ptr_override[name]
        pl = self.place(name)
        return f"pv_{name}" if pl == "private" else f"c_{name}"

    # -- reads / writes ---------------------------------------------------------

    def read(self, m: sdfg.Memlet, env: dict, depth: int) -> tuple[str, str]:
        if m.container in self.redirect:
            return self.redirect[m.container], TC[self.g.containers[m.container].dtype]
        c = self.cont(m.container)
        t = TC[c.dtype]
        pl = self.place(m.container)
        if pl == "reg":
            return f"r_{m.container}", t
        if pl == "colstage":  # staged column vector (rowpass prologue)
            self.spec.arg_index(("ptr", m.container))
            return f"rp_smem[{self.colstage[m.container]} + jl]", t
        if depth == 0 and m.container in self.stencil and self.spec.mode == "tma3":
            self.spec.checks.append((m.container, m.subset, env))
            offs = self._stencil_offsets(m, env)
            key = (m.container, offs)
            hit = self.cse.get(key)
            if hit is None:
                st = self.stencil[m.container]
                hit = self.fresh("sm")
                self.emit(f"const double {hit} = tsm_{m.container}[sl_{offs[0] - st['min'][0]} + "
                          f"(ly + {offs[1] - st['min'][1]}) * T3_SK + "
                          f"lx + {offs[2] - st['min'][2]}];")
                self.cse[key] = hit
            return hit, t
        idx = [symexpr.to_c(b, self.name_of(env)) for b, _, _ in m.subset]
        off = self.offset(m.container, idx)
        p = self.ptr(m.container)
        if depth > 0 or pl == "private":
            v = self.fresh("ld")
            o = self.fresh("off")
            size = f"sz_{m.container}"
            site = self._site(f"read {m.text}")
            self.emit(f"const b2_ll {o} = {off};")
            self.emit(f"const {CT[c.dtype]} {v} = b2_oob({o}, {size}, {site}, flag) ? "
                      f"({CT[c.dtype]})0 : {p}[{o}];")
            return v, t
        self.spec.checks.append((m.container, m.subset, env))
        if m.container not in self.written:
            key = (m.container, off)
            hit = self.cse.get(key)
            if hit is None:
                hit = self.fresh("ld")
                if self.hoist:
                    self.hoisted.append((hit, CT[c.dtype], f"{p}[{off}]"))
                    hit = f"{hit}[v]"
                else:
                    self.emit(f"const {CT[c.dtype]} {hit} = {p}[{off}];")
                self.cse[key] = hit
            return hit, t
        return f"{p}[{off}]", t

    def _site(self, desc: str) -> int:
        self.spec.uses_flag = True
        self.spec.sites.append(desc)
        return self.group.idx * 4096 + len(self.spec.sites) - 1

    def write(self, m: sdfg.Memlet, code: str, vt: str, env: dict, depth: int):
        if m.container in self.redirect and m.wcr is None:
            want = TC[self.g.containers[m.container].dtype]
            self.emit(f"{self.redirect[m.container]} = {scalar.cast(code, vt, want)};")
            return
        c = self.cont(m.container)
        ct = CT[c.dtype]
        want = TC[c.dtype]
        pl = self.place(m.container)
        val = scalar.cast(code, vt, want)
        if c.dtype == "i32":
            val = f"(int)({val})"
        if pl == "reg":
            tgt = f"r_{m.container}"
            if m.wcr is None:
                self.emit(f"{tgt} = {val};")
            else:
                self.emit(f"{tgt} = b2_op_{m.wcr}({tgt}, ({ct})({val}));")
            return
        if self.red is not None and m.wcr is not None and depth == 0:
            key = self._wkey(m, env)
            t = self.red.get(key)
            if t is None:
                idx = [symexpr.to_c(b, self.name_of(env)) for b, _, _ in m.subset]
                self.spec.checks.append((m.container, m.subset, env))
                t = {"acc": self.fresh("acc"), "ct": ct, "wcr": m.wcr, "cont": m.container,
                     "target": f"{self.ptr(m.container)}[{self.offset(m.container, idx)}]",
                     "exclusive": self.red_targets[key][1] == set(self.red_pout)}
                self.red[key] = t
            a = t["acc"]
            if self.red_full and t["exclusive"]:
                self.emit(f"{a} = b2_op_{m.wcr}({a}, ({ct})({val}));")
            else:
                # accumulator starts at the WCR identity (a data-dependent
                # first-value select here also hung under nvcc 12.9 / sm_100a)
                self.emit(f"{a} = b2_op_{m.wcr}({a}, ({ct})({val}));")
            return
        # subset may cover several elements: broadcast assignment
        loops = []
        idx = []
        for d, (b, e, s) in enumerate(m.subset):
            if b == e:
                idx.append(symexpr.to_c(b, self.name_of(env)))
            else:
                v = self.fresh("w")
                bb = symexpr.to_c(b, self.name_of(env))
                ee = symexpr.to_c(e, self.name_of(env))
                ss = symexpr.to_c(s, self.name_of(env))
                loops.append(f"for (b2_ll {v} = {bb}; {v} <= {ee}; {v} += {ss})")
                idx.append(v)
        for lp in loops:
            self.emit(lp + " {")
            self.ind += 2
        off = self.offset(m.container, idx)
        p = self.ptr(m.container)
        guarded = depth > 0 or loops or pl == "private"
        shared = (self.group.schedule == "parallel" and bool(self.group.params)
                  and pl == "memory")
        if guarded:
            o = self.fresh("off")
            site = self._site(f"write {m.text}")
            self.emit(f"const b2_ll {o} = {off};")
            self.emit(f"if (!b2_oob({o}, sz_{m.container}, {site}, flag)) {{")
            target = f"{p}[{o}]"
            self.ind += 2
        else:
            self.spec.checks.append((m.container, m.subset, env))
            target = f"{p}[{off}]"
        if m.wcr is None:
            self.emit(f"{target} = ({ct})({val});")
        elif shared:
            self.emit(f"b2_atomic_{m.wcr}(&{target}, ({ct})({val}));")
        else:
            self.emit(f"{target} = b2_op_{m.wcr}({target}, ({ct})({val}));")
        if guarded:
            self.ind -= 2
            self.emit("}")
        for _ in loops:
            self.ind -= 2
            self.emit("}")

    # -- body -------------------------------------------------------------------

    def tasklet(self, st: sdfg.State, t: sdfg.Tasklet, env: dict, depth: int):
        types: dict[str, str] = {}
        cname: dict[str, str] = {}
        self.emit(f"// tasklet {t.name} (node {t.id})")
        for e in st.in_edges(t):
            if e.memlet is None:
                continue
            code, ty = self.read(e.memlet, env, depth)
            v = self.fresh("in")
            cdt = CT[self.g.containers[e.memlet.container].dtype]
            self.emit(f"const {cdt} {v} = {code};")
            types[e.dst_conn] = ty
            cname[e.dst_conn] = v
        for _, code in t.code:
            for n in scalar.free_names(code):
                if n in types:
                    continue
                if n in env:
                    types[n] = "i"
                    cname[n] = env[n]
                elif n in self.g.containers:
                    raise P.PlanError(f"tasklet {t.name} reads container '{n}' without a memlet")
                else:
                    types[n] = "i"
                    cname[n] = self.sym(n)
        results: dict[str, tuple[str, str]] = {}
        for conn, code in t.code:
            c, ty = scalar.emit(code, types, lambda n: cname[n])
            v = self.fresh("o")
            self.emit(f"const {scalar.ctype(ty)} {v} = {c};")
            results[conn] = (v, ty)
        for e in st.out_edges(t):
            if e.memlet is None:
                continue
            key = e.src_conn if e.src_conn in results else t.outs[0]
            v, ty = results[key]
            self.write(e.memlet, v, ty, env, depth)

    def scope(self, st: sdfg.State, entry: sdfg.MapEntry, env: dict, depth: int):
        for c in P._scope_children(st, entry):
            if isinstance(c, sdfg.Tasklet):
                self.tasklet(st, c, env, depth)
            elif isinstance(c, sdfg.MapEntry):
                inner = dict(env)
                heads = []
                for p, (b, e, s) in c.params:
                    v = self.fresh(f"p_{p}")
                    bb = symexpr.to_c(b, self.name_of(inner))
                    ee = symexpr.to_c(e, self.name_of(inner))
                    ss = symexpr.to_c(s, self.name_of(inner))
                    heads.append(f"for (b2_ll {v} = {bb}; {v} <= {ee}; {v} += {ss})")
                    inner[p] = v
                for h in heads:
                    self.emit(h + " {")
                    self.ind += 2
                self.scope(st, c, inner, depth + 1)
                for _ in heads:
                    self.ind -= 2
                    self.emit("}")
            elif isinstance(c, sdfg.Library):
                self.library_in_scope(st, c, env, depth + 1)
            elif isinstance(c, (sdfg.Access, sdfg.MapExit)):
                pass
            else:
                raise P.PlanError(f"unsupported node {type(c).__name__} inside a map scope")

    def library_in_scope(self, st, n: sdfg.Library, env, depth):
        """REDUCE inside a map scope (doitgen): sequential in-thread loop with
        np.<op>.reduce semantics over the input subset (interp.py:461-473)."""
        if n.kind != "reduce" or n.attrs.get("axes") is not None:
            raise P.PlanError(f"library node '{n.kind}' inside a map scope is not supported")
        ins = [e for e in st.in_edges(n) if e.memlet is not None]
        outs = [e for e in st.out_edges(n) if e.memlet is not None]
        op = n.attrs.get("op", "add")
        m = ins[0].memlet
        c = self.cont(m.container)
        acc = self.fresh("acc")
        first = self.fresh("first")
        self.emit("{")
        self.ind += 2
        ident = {"add": "0.0", "mul": "1.0", "min": "b2_inf()", "max": "(-b2_inf())"}[op]
        self.emit(f"double {acc} = {ident}; bool {first} = true;")
        loops, idx = [], []
        for (b, e, s) in m.subset:
            v = self.fresh("r")
            loops.append(f"for (b2_ll {v} = {symexpr.to_c(b, self.name_of(env))}; "
                         f"{v} <= {symexpr.to_c(e, self.name_of(env))}; "
                         f"{v} += {symexpr.to_c(s, self.name_of(env))})")
            idx.append(v)
        for lp in loops:
            self.emit(lp + " {")
            self.ind += 2
        if self.place(m.container) == "reg":
            val = f"r_{m.container}"
        else:
            o = self.fresh("off")
            site = self._site(f"reduce read {m.text}")
            self.emit(f"const b2_ll {o} = {self.offset(m.container, idx)};")
            val = self.fresh("v")
            self.emit(f"const double {val} = b2_oob({o}, sz_{m.container}, {site}, flag) ? 0.0 : "
                      f"(double){self.ptr(m.container)}[{o}];")
        comb = {"add": f"{acc} + {val}", "mul": f"{acc} * {val}",
                "min": f"b2_npmin({acc}, {val})", "max": f"b2_npmax({acc}, {val})"}[op]
        self.emit(f"{acc} = {first} ? {val} : ({comb}); {first} = false;")
        for _ in loops:
            self.ind -= 2
            self.emit("}")
        for e in outs:
            self.write(e.memlet, acc, "f", env, depth)
        self.ind -= 2
        self.emit("}")
        _ = c

    # -- kernel -----------------------------------------------------------------

    def build(self) -> KernelSpec:
        grp = self.group
        spec = self.spec
        k = len(grp.params)
        # constant (non loop-assigned) ranges are baked into the source
        self.const_ranges = [_const_range(self.pl, r) for r in grp.ranges]
        if grp.schedule == "scalar":
            mode = "scalar"
        elif grp.schedule == "sequential":
            mode = "seq"
        else:
            mode = "flat"
            if k >= 2:
                last = self.const_ranges[-1]
                prev = self.const_ranges[-2]
                if last is not None and prev is not None and last[2] >= 16 and prev[2] >= 4:
                    mode = "tile2"
            if (mode == "tile2" and k == 3 and self.const_ranges[0] is not None
                    and self.const_ranges[0][2] >= 16):
                mode = "march"  # measured best for 3-D sweeps (heat_3d: 207 us vs 247 tile2)

        if (mode == "march" and TMA3 and not getattr(self.pl, "dynamic_p0", False)
                and all(r is not None and r[1] == 1 for r in self.const_ranges)
                and all(r[2] >= 8 for r in self.const_ranges)):
            st = self._stencil_analysis()
            if st and all(self.g.containers[c].dtype == "f64" for c in st):
                sts = next(iter(st.values()))
                if all(sts["max"][d] - sts["min"][d] <= 2 for d in range(3)):
                    self.stencil = st
                    mode = "tma3"
        force = os.environ.get("B2_FORCE_MODE")  # tuning knob: flat | tile2 | march
        if force and mode in ("flat", "tile2", "march") and k >= 1:
            if force == "march" and (k < 3 or any(r is None for r in self.const_ranges)):
                pass
            elif force != "tile2" or k >= 2:
                mode = force
        if mode != "tma3":
            self.stencil = {}
        if mode in ("flat", "tile2", "march") and CONTRACT_MODE and k >= 2:
            cp = self._contraction_plan()
            if cp is not None:
                spec.mode = "contract"
                sl = self._slide_plan(cp) if CONTRACT_SLIDE else None
                return self._contract_slide_kernel(cp, sl) if sl else self._contract_kernel(cp)
        if mode in ("flat", "tile2", "march") and REDUCE_MODE:
            rp = self._reduction_plan()
            if (rp is not None and ROWRED_MODE and ROWRED_CONTIG and rp[0] == [grp.params[-1]]
                    and math.prod(self.const_ranges[i][2] for i in range(k - 1)) >= ROWRED_CONTIG_MINROWS
                    and self._last_param_contiguous() and self._rowred_plan() is not None):
                # reducing over the contiguous dimension (the expanded GEMV
                # row dot A[i, :] . x) with rows enough for a warp each: a
                # thread per output reads rows strided by the row length, a
                # warp per row reads them coalesced
                rp = None
            if rp is not None:
                R, pout, targets = rp
                mode = "reduce"
                self.red = {}
                self.red_targets = targets
                self.red_pout = pout
                nout = 1
                for p in pout:
                    nout *= self.const_ranges[grp.params.index(p)][2]
                nred = 1
                for p in R:
                    nred *= self.const_ranges[grp.params.index(p)][2]
                self.red_full = nout >= 148 * 256 or nred <= 64
                self.red_R = R
        if mode in ("flat", "tile2", "march") and ROWRED_MODE:
            rp = self._rowred_plan()
            if rp is not None:
                R, pout, targets = rp
                mode = "rowred"
                self.red = {}
                self.red_targets = targets
                self.red_pout = pout
                self.red_full = False
                self.red_R = R
                if self.epi_group is not None and ROWRED_EPILOGUE:
                    self.epi = self._epilogue_plan(self.epi_group)
        if (mode == "tile2" and k == 2 and MARCH2
                and not getattr(self.pl, "dynamic_p0", False)
                and self.const_ranges[0][2] >= 4 * MARCH2_V
                and self.const_ranges[0][2] * self.const_ranges[1][2] <= (1 << 24)):
            mode = "march2"  # (reductions / row reductions / contractions keep theirs)
        spec.mode = mode
        # slab executors launch a map's chunk in pieces (boundary rows first,
        # interior overlapped with the halo exchange): keep dim 0's range a
        # runtime argument so one kernel serves every piece
        self.dyn0 = (bool(getattr(self.pl, "dynamic_p0", False)) and k >= 1
                     and mode in ("flat", "tile2", "march"))
        spec.dyn0 = self.dyn0
        vec = 1
        if mode == "tile2":
            vec = _pick_vec(self.const_ranges[-1][2])
            npts = 1
            for r in self.const_ranges:
                npts *= r[2] if r is not None else 1 << 30
            if npts <= (1 << 24):
                # small (L2-resident) sweeps: more threads beat longer rows
                # (jacobi_2d N=2000: 1.74 ms at vec 2 vs 1.83 at vec 4)
                vec = min(vec, 2)
        elif mode == "march":
            # 16 planes per thread measured 3 % faster on heat_3d N=400 (202 vs
            # 209 us); short or runtime dim-0 ranges (slabs) keep 8
            r0 = self.const_ranges[0]
            if self.dyn0:
                # slab executors: measured per-rank times at P=2/4/8 (heat_3d
                # N=400, scripts/scaling_projection.py) with the L2 prefetch
                # are best at 8 planes (6 without it)
                vec = SLAB_VEC
            else:
                vec = 16 if (r0 is not None and r0[2] >= 256) else 8
        elif mode == "march2":
            vec = MARCH2_V  # rows per thread
        elif mode == "tma3":
            vec = 2  # points per thread along the row (tile width <= 64)
        elif mode == "flat" and all(r is not None for r in self.const_ranges):
            total = 1
            for r in self.const_ranges:
                total *= r[2]
            vec = 4 if total >= 4 * 256 * 148 else 1
        if os.environ.get("B2_VEC"):
            vec = int(os.environ["B2_VEC"])
        spec.vec = vec
        spec.align = 0
        spec.block = {"scalar": (1, 1, 1), "seq": (1, 1, 1), "flat": (256, 1, 1),
                      "tile2": (32, TILE_BY, 1), "march": (SLAB_BX if self.dyn0 else MARCH_BX, MARCH_BY, 1), "reduce": (256, 1, 1),
                      "march2": (64, MARCH2_BY, 1),
                      "rowred": (256, 1, 1), "tma3": (32, TMA3_CW + 1, 1)}[mode]

        # containers written anywhere in this group: the rest are read-only
        self.written = set()
        self.read_set = set()
        for mem in grp.members:
            for a in self.pl.member_accesses(mem, grp.params):
                if a[1]:
                    self.written.add(a[0])
                else:
                    self.read_set.add(a[0])
        self.cse = {}
        # batch the read-only loads of all `vec` points of a thread ahead of
        # their arithmetic: memory-level parallelism without extra warps
        # flat / tile2: each thread's vec points issue their read-only loads
        # before the math (softmax's divide map 0.78 -> 0.64 ms; neutral on
        # jacobi_2d / go_fast).  march keeps program order: 16 planes x 7
        # hoisted loads per thread tripled heat_3d's time.
        self.hoist = mode in ("flat", "tile2") and vec > 1 and HOIST_TILES
        self.hoisted = []

        env = {p: f"p_{p}" for p in grp.params}
        if self.epi is not None:
            self.redirect = {T: f"tb_{T}[v]" for T in self.epi["T"]}
        body_lines_start = len(self.lines)
        self.ind = 6
        for mem in grp.members:
            menv = {mp: env[gp] for mp, gp in mem.rename.items()}
            if mem.tasklet is not None:
                self.tasklet(mem.state, mem.tasklet, menv, 0)
            else:
                self.scope(mem.state, mem.entry, menv, 0)
        body = self.lines[body_lines_start:]
        self.lines = self.lines[:body_lines_start]
        self.epi_body = []
        if self.epi is not None:
            # the epilogue map: reads of T from the row registers, of the
            # reduction targets from the (warp-reduced) accumulators
            B = self.epi["B"]
            for t in self.red.values():
                self.redirect[t["cont"]] = t["acc"]
            for mem in B.members:
                for (c, w, wcr, depth, pt) in self.pl.member_accesses(mem, B.params):
                    (self.written if w else self.read_set).add(c)
            benv = {bp: f"p_{ap}" for bp, ap in zip(B.params, grp.params)}
            start = len(self.lines)
            self.ind = 6
            for mem in B.members:
                menv = {mp: benv[gp] for mp, gp in mem.rename.items()}
                if mem.tasklet is not None:
                    self.tasklet(mem.state, mem.tasklet, menv, 0)
                else:
                    self.scope(mem.state, mem.entry, menv, 0)
            self.epi_body = self.lines[start:]
            self.lines = self.lines[:start]
            self.redirect = {}
            spec.epilogue = B.idx

        pro: list[str] = []
        nthr = spec.block[0] * spec.block[1] * spec.block[2]
        minb = f", {ROWRED_MINB}" if mode == "rowred" and ROWRED_MINB else ""
        if mode == "rowred" and self.epi is not None:
            # the row lives in registers (tb_*): fewer resident CTAs, no spills
            minb = f", {ROWRED_EPI_MINB}"
        pro.append(f'extern "C" __global__ void __launch_bounds__({max(256, nthr)}{minb}) '
                   f"{spec.name}(const __grid_constant__ B2Args a) {{")
        pro.append("  B2_PDL_ENTRY();")
        def _size(name):
            n = 1
            for x in self.shapes[name]:
                n *= x
            return n

        # small thread-private transients (e.g. a tiled WCR's stack
        # accumulator) live in a per-point local array, not in HBM scratch
        small_priv = [n for n in spec.containers
                      if self.place(n) == "private" and _size(n) <= SMALL_PRIVATE]
        for name in spec.containers:
            c = self.g.containers[name]
            pl = self.place(name)
            if pl == "reg":
                continue
            if name in small_priv:
                pro.append(f"  {CT[c.dtype]} pva_{name}[{_size(name)}];")
            else:
                base = self.arg(("ptr", name))
                ro = name not in self.written and pl == "memory"
                q = "const " if ro else ""
                pro.append(f"  {q}{CT[c.dtype]} *__restrict__ c_{name} = ({q}{CT[c.dtype]} *){base};")
            shape = self.shapes[name]
            st = _row_major(shape)
            for d in range(len(shape)):
                pro.append(f"  constexpr b2_ll st_{name}_{d} = {st[d]}LL;")
            n = 1
            for x in shape:
                n *= x
            pro.append(f"  constexpr b2_ll sz_{name} = {n}LL;")
        for s in spec.syms:
            if s in self.pl.fixed:
                pro.append(f"  constexpr b2_ll s_{s} = {int(self.pl.fixed[s])}LL;")
            else:
                pro.append(f"  const b2_ll s_{s} = {self.arg(('sym', s))};")
        pro.append(f"  int *flag = (int *){self.arg(('flag',))};")
        pro.append("  (void)flag;")
        for i in range(k):
            cr = self.const_ranges[i]
            if cr is not None and i == 0 and self.dyn0:
                # runtime start/length, compile-time stride: the compiler still
                # sees that consecutive i0 of one thread are adjacent planes
                pro.append(f"  const b2_ll rb0 = {self.arg(('rb', 0))};")
                pro.append(f"  constexpr b2_ll rs0 = {cr[1]}LL;")
                pro.append(f"  const b2_ll rl0 = {self.arg(('rl', 0))};")
            elif cr is not None:
                pro.append(f"  constexpr b2_ll rb{i} = {cr[0]}LL, rs{i} = {cr[1]}LL, rl{i} = {cr[2]}LL;")
            else:
                pro.append(f"  const b2_ll rb{i} = {self.arg(('rb', i))};")
                pro.append(f"  const b2_ll rs{i} = {self.arg(('rs', i))};")
                pro.append(f"  const b2_ll rl{i} = {self.arg(('rl', i))};")
        for n in small_priv:
            pro.append(f"  {CT[self.g.containers[n].dtype]} *__restrict__ pv_{n} = pva_{n};")
        privates = [n for n in spec.containers
                    if self.place(n) == "private" and n not in small_priv]
        if privates:
            pro.append("  const b2_ll tflat = ((b2_ll)blockIdx.x * blockDim.y + threadIdx.y) * "
                       "blockDim.x + threadIdx.x;")
            for n in privates:
                pro.append(f"  {CT[self.g.containers[n].dtype]} *__restrict__ pv_{n} = c_{n} + "
                           f"tflat * sz_{n};")
                spec.private[n] = 1
        regs = [n for n in spec.containers if self.place(n) == "reg"]

        def reg_decls(indent):
            out = [" " * indent + f"{CT[self.g.containers[n].dtype]} r_{n} = 0;" for n in regs]
            out += [" " * indent + f"for (int z = 0; z < {_size(n)}; ++z) pva_{n}[z] = 0;"
                    for n in small_priv]
            return out

        def shift(lines, by):
            return [(" " * by + ln) if by >= 0 else ln[-by:] for ln in lines]

        loop: list[str] = []
        if mode == "scalar":
            loop.append("  if (blockIdx.x == 0 && threadIdx.x == 0) {")
            loop += reg_decls(4)
            loop += shift(body, -2)
            loop.append("  }")
        elif mode == "seq":
            loop.append("  if (blockIdx.x == 0 && threadIdx.x == 0) {")
            for i, p in enumerate(grp.params):
                loop.append(f"  for (b2_ll i{i} = 0; i{i} < rl{i}; ++i{i}) {{")
                loop.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * i{i};")
            loop += reg_decls(4)
            loop += body
            for _ in grp.params:
                loop.append("  }")
            loop.append("  }")
        def vloop(header: list) -> list:
            """Per-thread loop over its `vec` points: phase 1 issues every
            hoisted read-only load of every point, phase 2 does the math."""
            out: list[str] = []
            if self.hoisted:
                for name, ct, _ in self.hoisted:
                    out.append(f"    {ct} {name}[{vec}];")
                out.append("#pragma unroll")
                out.append(f"    for (int v = 0; v < {vec}; ++v) {{")
                out += header
                for name, _, expr in self.hoisted:
                    out.append(f"    {name}[v] = {expr};")
                out.append("    }")
            out.append("#pragma unroll")
            out.append(f"    for (int v = 0; v < {vec}; ++v) {{")
            out += header
            out += reg_decls(4)
            out += shift(body, -2)
            out.append("    }")
            return out

        if mode == "flat":
            tot = " * ".join(f"rl{i}" for i in range(k))
            loop.append(f"  const b2_ll total = {tot};")
            loop.append(f"  for (b2_ll f0 = (b2_ll)blockIdx.x * blockDim.x * {vec}; f0 < total; "
                        f"f0 += (b2_ll)gridDim.x * blockDim.x * {vec}) {{")
            hdr = ["    const b2_ll f = f0 + (b2_ll)v * blockDim.x + threadIdx.x;",
                   "    if (f >= total) break;", "    b2_ll rem = f;"]
            for i in reversed(range(k)):
                p = grp.params[i]
                if i > 0:
                    hdr.append(f"    const b2_ll i{i} = rem % rl{i}; rem /= rl{i};")
                else:
                    hdr.append(f"    const b2_ll i{i} = rem;")
                hdr.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * i{i};")
            loop += vloop(hdr)
            loop.append("  }")
        elif mode == "tma3":
            loop += self._tma3_loop(reg_decls, shift(body, -2))
        elif mode == "reduce":
            loop += self._reduce_loop(self.red_R, self.red_pout, reg_decls, shift(body, -2))
        elif mode == "rowred":
            loop += self._rowred_loop(self.red_pout, reg_decls, shift(body, -2))
        elif mode == "tile2":
            x, y = k - 1, k - 2
            tw = 32 * vec
            ax = spec.align
            loop.append(f"  const b2_ll tiles_x = (rl{x} + {ax + tw - 1}) / {tw};")
            tby = spec.block[1]
            loop.append(f"  const b2_ll tiles_y = (rl{y} + {tby - 1}) / {tby};")
            outer = " * ".join(f"rl{i}" for i in range(k - 2)) or "1"
            loop.append(f"  const b2_ll nvb = tiles_x * tiles_y * ({outer});")
            loop.append("  for (b2_ll vb = blockIdx.x; vb < nvb; vb += gridDim.x) {")
            loop.append("    const b2_ll tx = vb % tiles_x; b2_ll rem = vb / tiles_x;")
            loop.append("    const b2_ll ty = rem % tiles_y; rem /= tiles_y;")
            for i in reversed(range(k - 2)):
                if i > 0:
                    loop.append(f"    const b2_ll i{i} = rem % rl{i}; rem /= rl{i};")
                else:
                    loop.append(f"    const b2_ll i{i} = rem;")
            loop.append(f"    const b2_ll i{y} = ty * {tby} + threadIdx.y;")
            loop.append(f"    if (i{y} >= rl{y}) continue;")
            if ax:
                hdr = [f"    const b2_ll i{x} = tx * {tw} + v * 32 + (b2_ll)threadIdx.x - {ax};",
                       f"    if (i{x} >= rl{x}) break;",
                       f"    if (i{x} < 0) continue;"]
            else:
                hdr = [f"    const b2_ll i{x} = tx * {tw} + v * 32 + threadIdx.x;",
                       f"    if (i{x} >= rl{x}) break;"]
            for i, p in enumerate(grp.params):
                hdr.append(f"    const b2_ll p_{p} = rb{i} + rs{i} * i{i};")
            if MARCH_FULL and vec > 1:
                loop.append(f"    if (tx * {tw} >= {ax} && tx * {tw} + {tw - ax} <= rl{x}) {{")
                loop += vloop([hdr[0]] + hdr[3 if ax else 2:])
                loop.append("    } else {")
                loop += vloop(hdr)
                loop.append("    }")
            else:
                loop += vloop(hdr)
            loop.append("  }")
        elif mode == "march2":
            # 64-column tiles of MARCH2_BY x vec rows: each thread walks `vec`
            # consecutive rows (unrolled), so a stencil's north / centre rows
            # come from the previous iterations' registers
            rows = spec.block[1] * vec
            loop.append("  const b2_ll tiles_x = (rl1 + 63) / 64;")
            loop.append(f"  const b2_ll tiles_y = (rl0 + {rows - 1}) / {rows};")
            loop.append("  for (b2_ll vb = blockIdx.x; vb < tiles_x * tiles_y; vb += gridDim.x) {")
            loop.append("    const b2_ll tx = vb % tiles_x, ty = vb / tiles_x;")
            loop.append("    const b2_ll i1 = tx * 64 + threadIdx.x;")
            loop.append("    if (i1 >= rl1) continue;")
            loop.append(f"    const b2_ll p_{grp.params[1]} = rb1 + rs1 * i1;")
            loop.append(f"    const b2_ll r0 = (ty * {spec.block[1]} + threadIdx.y) * {vec};")
            hdr = ["    const b2_ll i0 = r0 + v;", "    if (i0 >= rl0) break;",
                   f"    const b2_ll p_{grp.params[0]} = rb0 + rs0 * i0;"]
            if MARCH_FULL:
                loop.append(f"    if (r0 + {vec} <= rl0) {{")
                loop += vloop([hdr[0], hdr[2]])
                loop.append("    } else {")
                loop += vloop(hdr)
                loop.append("    }")
            else:
                loop += vloop(hdr)
            loop.append("  }")
        elif mode == "march":
            # 32 x 8 tiles over dims (k-2, k-1); each thread walks `vec`
            # consecutive indices of dim 0 (unrolled) so the compiler reuses the
            # overlapping dim-0 neighbours of a stencil from registers
            x, y = k - 1, k - 2
            by = MARCH_BY
            ax = spec.align
            bx = spec.block[0]
            loop.append(f"  const b2_ll tiles_x = (rl{x} + {ax + bx - 1}) / {bx};")
            loop.append(f"  const b2_ll tiles_y = (rl{y} + {by - 1}) / {by};")
            loop.append(f"  const b2_ll tiles_z = (rl0 + {vec - 1}) / {vec};")
            mid = " * ".join(f"rl{i}" for i in range(1, k - 2)) or "1"
            loop.append(f"  const b2_ll nvb = tiles_x * tiles_y * ({mid}) * tiles_z;")
            # plane tiles vary fastest (measured better than chunk-fastest order)
            loop.append("  for (b2_ll vb = blockIdx.x; vb < nvb; vb += gridDim.x) {")
            loop.append("    const b2_ll tx = vb % tiles_x; b2_ll rem = vb / tiles_x;")
            loop.append("    const b2_ll ty = rem % tiles_y; rem /= tiles_y;")
            for i in reversed(range(1, k - 2)):
                loop.append(f"    const b2_ll i{i} = rem % rl{i}; rem /= rl{i};")
            loop.append("    const b2_ll tz = rem;")
            if (SLAB_PREFETCH if self.dyn0 else MARCH_PREFETCH) and k == 3:
                loop += self._march_prefetch(vec, by, spec.align)
            loop.append(f"    const b2_ll i{y} = ty * {by} + threadIdx.y;")
            if ax:
                loop.append(f"    const b2_ll i{x} = tx * {bx} + (b2_ll)threadIdx.x - {ax};")
                loop.append(f"    if (i{y} >= rl{y} || i{x} >= rl{x} || i{x} < 0) continue;")
            else:
                loop.append(f"    const b2_ll i{x} = tx * {bx} + threadIdx.x;")
                loop.append(f"    if (i{y} >= rl{y} || i{x} >= rl{x}) continue;")
            for i in range(1, k):
                loop.append(f"    const b2_ll p_{grp.params[i]} = rb{i} + rs{i} * i{i};")
            hdr = [f"    const b2_ll i0 = tz * {vec} + v;", "    if (i0 >= rl0) break;",
                   f"    const b2_ll p_{grp.params[0]} = rb0 + rs0 * i0;"]
            if MARCH_FULL and vec > 1:
                # full plane tiles take a branch-free copy of the unrolled
                # loop so loads of later planes can issue before earlier math
                loop.append(f"    if (tz * {vec} + {vec} <= rl0) {{")
                loop += vloop([hdr[0], hdr[2]])
                loop.append("    } else {")
                loop += vloop(hdr)
                loop.append("    }")
            else:
                loop += vloop(hdr)
            loop.append("  }")
        src = [f"// generated by paper_2107_00555_b200.codegen for state "
               f"'{grp.state.label}', group of {len(grp.members)} scope(s), mode {mode}, vec {vec}"]
        if spec.tmaps:
            src.append("struct __align__(64) B2TMap { unsigned long long v[16]; };")
            src.append("struct B2Args { B2TMap tm[%d]; long long w[%d]; };"
                       % (len(spec.tmaps), max(1, len(spec.args))))
        else:
            src.append("struct B2Args { long long w[%d]; };" % max(1, len(spec.args)))
        fin = self._reduce_fin(pro) if mode == "reduce" and getattr(spec, "red_fin", None) else []
        npts = 1
        for r in self.const_ranges:
            npts *= r[2] if r is not None else 1 << 40
        spec.pdl = ((MARCH_PDL and mode in ("march", "tma3")) or (TILE_PDL and mode == "tile2")
                    or (MARCH2_PDL and mode == "march2")
                    or (SMALL_PDL and mode in ("flat", "reduce", "scalar")
                        and npts <= SMALL_PDL_POINTS)) and not self.dyn0
        if spec.pdl:
            # programmatic dependent launch: wait for the previous sweep's
            # grid at entry, trigger our dependents only after this CTA's
            # stores, so the next sweep launches into this one's tail
            pro.insert(pro.index("  B2_PDL_ENTRY();") + 1,
                       '  asm volatile("griddepcontrol.wait;" ::: "memory");')
            loop.append('  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");')
        spec.source = "\n".join(src + pro + loop + ["}"] + fin) + "\n"
        return spec


def _row_major(shape) -> list[int]:
    st = [1] * len(shape)
    acc = 1
    for d in range(len(shape) - 1, -1, -1):
        st[d] = acc
        acc *= shape[d]
    return st


def _pick_vec(n: int) -> int:
    """Points per thread along the innermost parameter: the largest of 4/2/1
    whose 32*vec-wide tiles waste at most 12% of the row."""
    for v in (4, 2):
        tw = 32 * v
        waste = (-(-n // tw) * tw - n) / max(1, n)
        if waste <= 0.13:
            return v
    return 1


def _const_range(planner: P.Planner, rng):
    b, e, s = rng
    try:
        env = dict(planner.fixed)
        bv, ev, sv = (symexpr.evaluate(x, env) for x in (b, e, s))
    except KeyError:
        return None
    if sv < 1:
        return None
    return bv, sv, max(0, (ev - bv) // sv + 1)


def point_function(planner: P.Planner, group: P.MapGroup, shapes: dict, fname: str,
                   env: dict, regs: dict, arg_base: int, signature: str, ret: str,
                   colstage: dict | None = None):
    """Emit the per-point body of ``group`` as a __device__ function (used to
    inline an elementwise map into another family, e.g. the rowpass
    prologue).  ``env`` maps group params to C expressions; ``regs`` maps
    containers to register names that replace their memory accesses."""
    gen = _Gen(planner, group, shapes, fname)
    gen.arg_base = arg_base
    gen.place_override = {c: "reg" for c in regs}
    gen.colstage = dict(colstage or {})
    for c in gen.colstage:
        gen.place_override[c] = "colstage"
    for mem in group.members:
        for a in planner.member_accesses(mem, group.params):
            if a[1]:
                gen.written.add(a[0])
    gen.ind = 2
    for mem in group.members:
        menv = {mp: env[gp] for mp, gp in mem.rename.items()}
        if mem.tasklet is not None:
            gen.tasklet(mem.state, mem.tasklet, menv, 0)
        else:
            gen.scope(mem.state, mem.entry, menv, 0)
    body = gen.lines
    decl = []
    for name in gen.spec.containers:
        if name in regs or name in gen.colstage:
            continue
        c = planner.g.containers[name]
        ro = name not in gen.written
        q = "const " if ro else ""
        decl.append(f"  {q}{CT[c.dtype]} *__restrict__ c_{name} = ({q}{CT[c.dtype]} *){gen.arg(('ptr', name))};")
        st = _row_major(shapes[name])
        for d in range(len(st)):
            decl.append(f"  constexpr b2_ll st_{name}_{d} = {st[d]}LL;")
        n = 1
        for x in shapes[name]:
            n *= x
        decl.append(f"  constexpr b2_ll sz_{name} = {n}LL;")
    for sname in gen.spec.syms:
        if sname in planner.fixed:
            decl.append(f"  constexpr b2_ll s_{sname} = {int(planner.fixed[sname])}LL;")
        else:
            raise P.PlanError("loop-assigned symbol in a fused prologue")
    if gen.spec.uses_flag:
        raise P.PlanError("guarded accesses in a fused prologue")
    src = [f"__device__ __forceinline__ {signature} {{"]
    src += decl
    src += [f"  {CT[planner.g.containers[c].dtype]} r_{c} = {r};" for c, r in regs.items()]
    src += body
    src += [f"  return {ret};", "}"]
    gen.spec.source = "\n".join(src) + "\n"
    return gen.spec


def generate_region(planner: P.Planner, reg, shapes: dict, name: str) -> KernelSpec:
    """One kernel for a device loop region (loops.py): parallel loops over
    threads, the rest of the nest as structured sequential C per thread.
    Every memory access inside is device-guarded (depth 1) because its index
    depends on loop symbols the host does not enumerate."""
    from . import loops as LP

    loops_all = LP.find_loops(planner)
    par_vars = [l.var for l in reg.par]
    dummy = P.MapGroup("map", planner.g.states[0], params=list(par_vars),
                       ranges=[], schedule="parallel" if par_vars else "scalar")
    dummy.idx = reg.idx
    gen = _Gen(planner, dummy, shapes, name)
    assigned = LP.assigned_symbols(planner, reg) - set(par_vars)
    sym_types = {}

    def name_of(n):
        return gen.sym(n)

    def cond_c(c):
        types = {n: "i" for n in scalar.free_names(c)}
        for n in types:
            gen.sym(n)
        code, t = scalar.emit(c, types, lambda n: f"s_{n}")
        return scalar.cast(code, t, "b")

    blockreg = bool(getattr(reg, "block", False))

    for c in getattr(reg, "private", ()):
        gen.place_override[c] = "private"  # per-iteration local copy (loops._privatisable)

    def emit_ops(h):
        for op in planner.ops[h]:
            if isinstance(op, P.LibOp) and op.node is not None and op.node.kind == "reduce":
                gen.library_in_scope(op.state, op.node, {}, 1)  # sequential, in-thread
                continue
            if not isinstance(op, P.MapGroup):
                raise P.PlanError("non-map op inside a device loop region")
            if blockreg:
                emit_block_group(op)
                continue
            for mem in op.members:
                if mem.tasklet is not None:
                    gen.tasklet(mem.state, mem.tasklet, {}, 1)
                    continue
                env = {}
                heads = []
                for p, (b, e, s) in mem.entry.params:
                    v = gen.fresh(f"p_{p}")
                    heads.append(f"for (b2_ll {v} = {symexpr.to_c(b, gen.name_of(env))}; "
                                 f"{v} <= {symexpr.to_c(e, gen.name_of(env))}; "
                                 f"{v} += {symexpr.to_c(s, gen.name_of(env))})")
                    env[p] = v
                for hd in heads:
                    gen.emit(hd + " {")
                    gen.ind += 2
                gen.scope(mem.state, mem.entry, env, 1)
                for _ in heads:
                    gen.ind -= 2
                    gen.emit("}")

    def emit_block_group(op):
        """Block region: a top-level tasklet group runs on thread 0; a map
        group's points are spread over the CTA's threads, each point running
        every member in order (the fused members share its op-local
        registers, as in the group's own kernel); a barrier orders the op
        before the next (block-scope visibility of its global writes)."""
        if op.schedule != "parallel":
            gen.emit("if (threadIdx.x == 0) {")
            gen.ind += 2
            for mem in op.members:
                gen.tasklet(mem.state, mem.tasklet, {}, 1)
            gen.ind -= 2
            gen.emit("}")
            gen.emit("__syncthreads();")
            return
        ns = []
        gen.emit("{")
        gen.ind += 2
        for p, (b, e, s_) in zip(op.params, op.ranges):
            bb, ee, ss = (symexpr.to_c(x, gen.name_of({})) for x in (b, e, s_))
            n, v0, st = gen.fresh(f"bn_{p}"), gen.fresh(f"bb_{p}"), gen.fresh(f"bs_{p}")
            gen.emit(f"const b2_ll {v0} = {bb}, {st} = {ss};")
            gen.emit(f"const b2_ll {n} = (({ee}) - {v0}) / {st} + 1;")
            ns.append((p, n, v0, st))
        tot = " * ".join(f"({n} > 0 ? {n} : 0)" for _, n, _, _ in ns) or "1"
        bf = gen.fresh("bf")
        gen.emit(f"for (b2_ll {bf} = threadIdx.x; {bf} < {tot}; {bf} += blockDim.x) {{")
        gen.ind += 2
        rem = gen.fresh("brem")
        gen.emit(f"b2_ll {rem} = {bf}; (void){rem};")
        gvar = {}
        for p, n, v0, st in reversed(ns):
            v = gen.fresh(f"p_{p}")
            gen.emit(f"const b2_ll {v} = {v0} + {st} * ({rem} % {n}); {rem} /= {n};")
            gvar[p] = v
        for mem in op.members:
            env = {mp: gvar[gp] for mp, gp in mem.rename.items()}
            gen.scope(mem.state, mem.entry, env, 1)
        gen.ind -= 2
        gen.emit("}")
        gen.ind -= 2
        gen.emit("}")
        gen.emit("__syncthreads();")

    def follow(t):
        for k, v in t.assignments.items():
            if k in par_vars:
                continue  # parallel loop variables come from the thread index
            gen.emit(f"s_{k} = {symexpr.to_c(v, name_of)};")

    def fold_info(L):
        """An inner loop that only folds ``C[idx] = max|min(C[idx], E(l))``
        or ``C[idx] = C[idx] + E(l)`` (idx independent of the loop variable,
        E reads anything but C), optionally after tasklets that only set
        op-local registers E reads (go_fast: ``e2 = exp(2 a[i, i])``).  The
        add fold re-associates the sum (within the rel_err 1e-12 contract;
        max / min folds are exact)."""
        if L.step <= 0 or L.body != {L.body_entry}:
            return None
        c = L.cond
        if not (isinstance(c, tuple) and c[0] == "bin" and c[1] in ("<", "<=")
                and c[2] == ("ref", L.var) and L.var not in scalar.free_names(c[3])):
            return None
        ops = planner.ops.get(L.body_entry, [])
        if len(ops) != 1 or not isinstance(ops[0], P.MapGroup):
            return None
        mems = ops[0].members
        if any(m.tasklet is None for m in mems):
            return None
        pre, mem = mems[:-1], mems[-1]
        for m in pre:  # helper tasklets: single statements into op-local registers
            outs_ = [e for e in m.state.out_edges(m.tasklet) if e.memlet is not None]
            if (len(m.tasklet.code) != 1 or len(outs_) != 1 or outs_[0].memlet.wcr is not None
                    or gen.place(outs_[0].memlet.container) != "reg"):
                return None
        t = mem.tasklet
        if len(t.code) != 1:
            return None
        outs = planner.g.out_transitions(planner.chain_end[L.body_entry])
        if len(outs) != 1 or outs[0].dst != L.guard or set(outs[0].assignments) != {L.var}:
            return None
        st = mem.state
        oe = [e for e in st.out_edges(t) if e.memlet is not None]
        ie = [e for e in st.in_edges(t) if e.memlet is not None]
        if len(oe) != 1 or oe[0].memlet.wcr is not None:
            return None
        om = oe[0].memlet
        if (planner.g.containers[om.container].dtype != "f64"
                or gen.place(om.container) == "reg"
                or any(L.var in symexpr.free_symbols(x) for d in om.subset for x in d)):
            return None
        code = t.code[0][1]
        if isinstance(code, tuple) and code[0] == "call" and code[1] in ("max", "min") \
                and len(code[2]) == 2:
            kind, (a0, a1) = code[1], code[2]
        elif isinstance(code, tuple) and code[0] == "bin" and code[1] == "+":
            kind, a0, a1 = "add", code[2], code[3]
        else:
            return None
        accs = [e for e in ie if e.memlet.container == om.container]
        if len(accs) != 1 or accs[0].memlet.text != om.text:
            return None
        acc_conn = accs[0].dst_conn
        if a0 == ("ref", acc_conn):
            expr = a1
        elif a1 == ("ref", acc_conn):
            expr = a0
        else:
            return None
        if acc_conn in scalar.free_names(expr):
            return None
        return {"op": kind, "state": st, "t": t, "acc": accs[0], "out": oe[0], "pre": pre,
                "others": [e for e in ie if e is not accs[0]], "expr": expr}

    def emit_fold(L, fi):
        """Warp-cooperative fold: lanes take every 32nd trip, combine with a
        fixed xor tree, lane 0 folds into C once (max/min are exact, so the
        result equals the sequential loop's for non-NaN data)."""
        op = {"max": "b2_pymax", "min": "b2_pymin", "add": "b2_op_add"}[fi["op"]]
        ident = {"max": "(-b2_inf())", "min": "b2_inf()", "add": "0.0"}[fi["op"]]
        cond = cond_c(L.cond)
        fa, fl, ran = gen.fresh("fold"), gen.fresh("fl"), gen.fresh("ran")
        gen.emit("{")
        gen.ind += 2
        # trip count of `var < B` / `var <= B` from the current value
        cb, _ = scalar.emit(L.cond[3], {n: "i" for n in scalar.free_names(L.cond[3])},
                            lambda n: f"s_{gen.sym(n)[2:]}")
        trip, fbase = gen.fresh("trip"), gen.fresh("fbase")
        extra = 1 if L.cond[1] == "<=" else 0
        gen.emit(f"const bool {ran} = {cond};")
        gen.emit(f"const b2_ll {trip} = {ran} ? ((b2_ll)({cb}) + {extra} - s_{L.var} + "
                 f"{L.step - 1}) / {L.step} : 0;")
        gen.emit(f"const b2_ll {fbase} = s_{L.var};")
        # reads affine in the loop variable: guard the first and last trip once
        # (device error flag as usual) so the loop body issues plain loads
        fi["checked"] = {}
        ok = gen.fresh("inb")
        gen.emit(f"bool {ok} = true;")
        for e in fi["others"]:
            m = e.memlet
            if gen.place(m.container) == "reg" or any(
                    symexpr.affine(b, tuple(symexpr.free_symbols(b)), {}) is None
                    for b, _, _ in m.subset):
                continue
            fi["checked"][id(e)] = True
            for at in (f"{fbase}", f"{fbase} + ({trip} - 1) * {L.step}"):
                idx = []
                gen.emit("{")
                gen.emit(f"  const b2_ll s_{L.var} = {at};")
                idx = [symexpr.to_c(b, gen.name_of({})) for b, _, _ in m.subset]
                site = gen._site(f"read {m.text}")
                gen.emit(f"  if ({trip} > 0 && b2_oob({gen.offset(m.container, idx)}, "
                         f"sz_{m.container}, {site}, flag)) {ok} = false;")
                gen.emit("}")
        gen.emit(f"double {fa} = {ident};")
        gen.emit(f"#pragma unroll {FOLD_UNROLL}")
        gen.emit(f"for (b2_ll {fl} = lane; {ok} && {fl} < {trip}; {fl} += 32) {{")
        gen.ind += 2
        gen.emit(f"const b2_ll s_{L.var} = {fbase} + {fl} * {L.step};")
        for m in fi["pre"]:  # helper registers (lane-private)
            gen.tasklet(m.state, m.tasklet, {}, 1)
        types, cname = {}, {}
        for e in fi["others"]:
            m = e.memlet
            cdt = CT[planner.g.containers[m.container].dtype]
            if fi["checked"].get(id(e)):
                # bounds proven at both ends of the trip range: plain load
                idx = [symexpr.to_c(b, gen.name_of({})) for b, _, _ in m.subset]
                code = f"{gen.ptr(m.container)}[{gen.offset(m.container, idx)}]"
                ty = TC[planner.g.containers[m.container].dtype]
            else:
                code, ty = gen.read(m, {}, 1)
            v = gen.fresh("in")
            gen.emit(f"const {cdt} {v} = {code};")
            types[e.dst_conn] = ty
            cname[e.dst_conn] = v
        for n in scalar.free_names(fi["expr"]):
            if n not in types:
                types[n] = "i"
                cname[n] = gen.sym(n)
        ec, et = scalar.emit(fi["expr"], types, lambda n: cname[n])
        gen.emit(f"{fa} = {op}({fa}, (double)({scalar.cast(ec, et, 'f')}));")
        gen.ind -= 2
        gen.emit("}")
        gen.emit(f"for (int o = 16; o > 0; o >>= 1) {fa} = {op}({fa}, "
                 f"__shfl_xor_sync(0xffffffffu, {fa}, o));")
        gen.emit(f"if (lane == 0 && {ran}) {{")
        gen.ind += 2
        ac, at = gen.read(fi["acc"].memlet, {}, 1)
        av = gen.fresh("acc")
        gen.emit(f"const double {av} = {ac};")
        gen.write(fi["out"].memlet, f"{op}({av}, {fa})", "f", {}, 1)
        gen.ind -= 2
        gen.emit("}")
        gen.emit("__syncwarp();")
        # the loop variable's exit value, in closed form (a counting loop
        # here cost every lane `trip` serial iterations)
        gen.emit(f"s_{L.var} = {fbase} + {trip} * {L.step};")
        gen.ind -= 2
        gen.emit("}")

    warp_mode = False
    if reg.par and FOLD_MODE and not blockreg:
        for h in reg.heads:
            if h in loops_all and h != reg.loop.guard and loops_all[h] not in reg.par \
                    and fold_info(loops_all[h]) is not None:
                warp_mode = True
    root_fold = None
    if not reg.par and FOLD_MODE and not blockreg:
        # the whole region is one fold loop (go_fast raw's trace): one warp
        root_fold = fold_info(reg.loop)
        warp_mode = root_fold is not None

    def block(cur, stop):
        guard_budget = 0
        while cur != stop:
            guard_budget += 1
            if guard_budget > 10000:
                raise P.PlanError("unstructured control flow in loop region")
            if cur in loops_all and cur in reg.heads:
                L = loops_all[cur]
                fi = fold_info(L) if warp_mode else None
                if fi is not None:
                    emit_fold(L, fi)
                    follow(L.t_out)
                    cur = L.exit
                    continue
                gen.emit(f"while ({cond_c(L.cond)}) {{")
                gen.ind += 2
                follow(L.t_in)
                block(L.body_entry, L.guard)
                gen.ind -= 2
                gen.emit("}")
                follow(L.t_out)
                cur = L.exit
                continue
            if warp_mode:  # lane 0 runs the plain code, the warp the folds
                gen.emit("if (lane == 0) {")
                gen.ind += 2
                emit_ops(cur)
                gen.ind -= 2
                gen.emit("}")
                gen.emit("__syncwarp();")
            else:
                emit_ops(cur)
            outs = planner.g.out_transitions(planner.chain_end[cur])
            if len(outs) != 1:
                raise P.PlanError("branching inside a device loop region")
            follow(outs[0])
            cur = outs[0].dst

    gen.ind = 6
    if reg.par:
        inner = reg.par[-1]
        follow(inner.t_in)
        block(inner.body_entry, inner.guard)
    elif root_fold is not None:
        emit_fold(reg.loop, root_fold)
    else:
        root = reg.loop
        gen.emit(f"while ({cond_c(root.cond)}) {{")
        gen.ind += 2
        follow(root.t_in)
        block(root.body_entry, root.guard)
        gen.ind -= 2
        gen.emit("}")
    body = gen.lines
    spec = gen.spec
    nthr = 256
    if blockreg:
        most = 1
        for h in reg.heads:
            for op in planner.ops[h]:
                if isinstance(op, P.MapGroup) and op.schedule == "parallel":
                    n = 1
                    for r in op.ranges:
                        n *= _const_range(planner, r)[2]
                    most = max(most, n)
        nthr = min(1024, max(64, -(-most // 32) * 32))
    pro = [f'extern "C" __global__ void __launch_bounds__({nthr}) {name}'
           "(const __grid_constant__ B2Args a) {", "  B2_PDL_ENTRY();"]
    for cname in spec.containers:
        c = planner.g.containers[cname]
        if gen.place(cname) == "reg":
            continue
        pro.append(f"  {CT[c.dtype]} *__restrict__ c_{cname} = ({CT[c.dtype]} *){gen.arg(('ptr', cname))};")
        st = _row_major(shapes[cname])
        for d in range(len(st)):
            pro.append(f"  constexpr b2_ll st_{cname}_{d} = {st[d]}LL;")
        n = 1
        for x in shapes[cname]:
            n *= x
        pro.append(f"  constexpr b2_ll sz_{cname} = {n}LL;")
    pro.append(f"  int *flag = (int *){gen.arg(('flag',))};")
    pro.append("  (void)flag;")
    npar = gen.arg(("npar",))
    pro.append(f"  const b2_ll NPAR = {npar};")
    for k, l in enumerate(reg.par):
        pro.append(f"  const b2_ll pb{k} = {gen.arg(('pb', k))}, ps{k} = {gen.arg(('ps', k))}, "
                   f"pn{k} = {gen.arg(('pn', k))};")
    if blockreg:  # one CTA, every thread walks the whole nest
        loop = ["  if (blockIdx.x != 0) return;", "  {", "    b2_ll rem = 0; (void)rem;"]
    elif warp_mode:  # one warp per parallel iteration
        loop = ["  const int lane = threadIdx.x & 31;",
                "  for (b2_ll f = ((b2_ll)blockIdx.x * blockDim.x + threadIdx.x) >> 5; f < NPAR; "
                "f += ((b2_ll)gridDim.x * blockDim.x) >> 5) {", "    b2_ll rem = f; (void)rem;"]
    else:
        loop = ["  for (b2_ll f = (b2_ll)blockIdx.x * blockDim.x + threadIdx.x; f < NPAR; "
                "f += (b2_ll)gridDim.x * blockDim.x) {", "    b2_ll rem = f; (void)rem;"]
    for k in reversed(range(len(reg.par))):
        loop.append(f"    const b2_ll s_{reg.par[k].var} = pb{k} + ps{k} * (rem % pn{k}); "
                    f"rem /= pn{k};")
    for s in spec.syms:
        if s in par_vars:
            continue
        if s in assigned:
            loop.append(f"    b2_ll s_{s} = {gen.arg(('sym', s))};")
        elif s in planner.fixed:
            loop.append(f"    constexpr b2_ll s_{s} = {int(planner.fixed[s])}LL;")
        else:
            loop.append(f"    const b2_ll s_{s} = {gen.arg(('sym', s))};")
    for cname in spec.containers:
        if gen.place(cname) == "reg":
            loop.append(f"    {CT[planner.g.containers[cname].dtype]} r_{cname} = 0;")
        elif gen.place(cname) == "private":
            ct = CT[planner.g.containers[cname].dtype]
            loop.append(f"    {ct} pva_{cname}[sz_{cname}];")
            loop.append(f"    {ct} *__restrict__ pv_{cname} = pva_{cname};")
    loop += [ln[2:] for ln in body]
    loop.append("  }")
    spec.source = "\n".join(
        [f"// generated by paper_2107_00555_b200.codegen: device loop region at "
         f"'{reg.loop.guard}' ({len(reg.par)} parallel loop(s))",
         "struct B2Args { long long w[%d]; };" % max(1, len(spec.args))] + pro + loop + ["}"]) + "\n"
    spec.mode = "region"
    spec.block = (nthr, 1, 1)
    spec.params = []
    spec.warp = warp_mode
    spec.block_region = blockreg
    return spec


def generate(planner: P.Planner, group: P.MapGroup, shapes: dict, name: str,
             init_const: dict | None = None, epilogue=None) -> KernelSpec:
    gen = _Gen(planner, group, shapes, name)
    gen.init_const = dict(init_const or {})
    gen.epi_group = epilogue
    spec = gen.build()
    spec.params = list(group.params)
    # reduction targets (container, point key) -> (exclusive, C type), for
    # the executor's init-map fusion
    spec.red_targets = {}
    if gen.red:
        for t in gen.red.values():
            spec.red_targets[t["cont"]] = spec.red_targets.get(t["cont"], []) + [
                (t["exclusive"], t["ct"])]
        spec.red_points = list(gen.red_targets)
    # args block decoded positionally; fix the struct size after all args known
    lines = spec.source.split("\n")
    k = next(i for i, ln in enumerate(lines) if ln.startswith("struct B2Args"))
    if spec.tmaps:
        lines[k] = "struct B2Args { B2TMap tm[%d]; long long w[%d]; };" % (
            len(spec.tmaps), max(1, len(spec.args)))
    else:
        lines[k] = "struct B2Args { long long w[%d]; };" % max(1, len(spec.args))
    spec.source = "\n".join(lines)
    return spec


# ---------------------------------------------------------------------------
# host-side launch recipe


def range_values(group: P.MapGroup, env: dict) -> list[tuple[int, int, int]]:
    out = []
    for b, e, s in group.ranges:
        bv = symexpr.evaluate(b, env)
        ev = symexpr.evaluate(e, env)
        sv = symexpr.evaluate(s, env)
        if sv < 1:
            raise ValueError(f"stride {sv} < 1 in map range")
        out.append((bv, sv, max(0, (ev - bv) // sv + 1)))
    return out


def launch_geometry(spec: KernelSpec, rl: list[int]) -> tuple[tuple, tuple]:
    if spec.mode in ("scalar", "seq"):
        return (1, 1, 1), (1, 1, 1)
    if spec.mode == "flat":
        total = 1
        for v in rl:
            total *= v
        blocks = max(1, min((total + 256 * spec.vec - 1) // (256 * spec.vec), MAX_BLOCKS * 8))
        if spec.private:
            blocks = max(1, min(blocks, MAX_BLOCKS))
        return (blocks, 1, 1), (256, 1, 1)
    k = len(rl)
    if spec.mode in ("reduce", "rowred"):
        n = getattr(spec, "red_threads", 1)
        return (max(1, min(-(-n // 256), MAX_BLOCKS * 8)), 1, 1), (256, 1, 1)
    if spec.mode == "tma3":
        return (spec.grid_cap, 1, 1), spec.block
    if spec.mode == "contract":
        c = spec.contract
        tiles = c.get("tiles_m", -(-c["M"] // c.get("TM", 128))) * -(-c["N"] // c["TN"])
        return (max(1, min(tiles, 148 * 8)), 1, 1), (256, 1, 1)
    if spec.mode == "march2":
        rows = spec.block[1] * spec.vec
        nvb = -(-rl[1] // 64) * -(-rl[0] // rows)
        return (max(1, min(nvb, MAX_BLOCKS * 8)), 1, 1), (64, spec.block[1], 1)
    if spec.mode == "march":
        bx, by = spec.block[0], spec.block[1]
        nvb = -(-(rl[k - 1] + spec.align) // bx) * -(-rl[k - 2] // by) * -(-rl[0] // spec.vec)
        for v in rl[1: k - 2]:
            nvb *= v
        blocks = max(1, min(nvb, MAX_BLOCKS * 8))
        if spec.private:
            blocks = max(1, min(blocks, MAX_BLOCKS))
        return (blocks, 1, 1), (bx, by, 1)
    tw = 32 * spec.vec
    tby = spec.block[1]
    tiles = ((rl[k - 1] + spec.align + tw - 1) // tw) * ((rl[k - 2] + tby - 1) // tby)
    for v in rl[: k - 2]:
        tiles *= v
    blocks = max(1, min(tiles, MAX_BLOCKS * 8))
    if spec.private:
        blocks = max(1, min(blocks, MAX_BLOCKS))
    return (blocks, 1, 1), (32, tby, 1)


def pack_args(spec: KernelSpec, env: dict, rvals, ptrs: dict, strides: dict, sizes: dict,
              scratch: dict, flag_ptr: int) -> bytes:
    vals = []
    for d in spec.args:
        k = d[0]
        if k == "ptr":
            vals.append(scratch[d[1]] if d[1] in scratch else ptrs[d[1]])
        elif k == "stride":
            vals.append(strides[d[1]][d[2]])
        elif k == "size":
            vals.append(sizes[d[1]])
        elif k == "sym":
            vals.append(int(env[d[1]]))
        elif k == "flag":
            vals.append(flag_ptr)
        elif k == "rb":
            vals.append(rvals[d[1]][0])
        elif k == "rs":
            vals.append(rvals[d[1]][1])
        elif k == "rl":
            vals.append(rvals[d[1]][2])
        else:
            raise AssertionError(d)
    if not vals:
        vals = [0]
    blob = struct.pack(f"<{len(vals)}q", *[v if v < (1 << 63) else v - (1 << 64) for v in vals])
    if spec.tmaps:
        from . import runtime as rt

        maps = b"".join(rt.tensor_map_f64(scratch[c] if c in scratch else ptrs[c],
                                          strides_shape(strides[c], sizes[c]), box)
                        for c, box in spec.tmaps)
        blob = maps + blob
    return blob


def strides_shape(st: list, size: int) -> tuple:
    """Row-major shape from row-major element strides and the element count."""
    shape = []
    prev = size
    for t in st:
        shape.append(prev // t)
        prev = t
    return tuple(shape)
