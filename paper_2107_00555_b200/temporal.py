"""Temporal pairing of two consecutive stencil sweeps into one HBM pass.

heat_3d's time step is two 3-D sweeps, ``X = f(Y)`` then ``Y = g(X)``
(Appendix B; each sweep is one fused map group after plan.py).  Run as two
kernels, every step streams Y in, X out, X in and Y out.  The paired kernel
marches a CTA tile along the outer dimension: each plane of X the tile's
``g`` needs (tile plus its halo) is produced by evaluating ``f`` — the same
tasklet chain, in the same order, so the values are bitwise identical — into
a shared-memory plane ring, written to HBM once by the CTA that owns it, and
``g`` then reads its whole stencil from the ring.  X is never re-read from
HBM (only its untouched boundary is).

``g`` writes Y while other CTAs still read Y's old values to evaluate ``f``
on their halos, so the pair writes into a second buffer (``Y#alt``) and the
executor swaps the two afterwards (machine.py): every step moves Y in, X
out and Y out — 3 array passes instead of 4.

Legality (``pair_info``), all checked on the planner's access sites:
  * both groups parallel, 3 parameters, identical constant unit-stride
    ranges, not inside a device loop region;
  * ``f`` writes exactly one memory container X (others are registers), at
    a single point ``p + o`` per iteration; ``g`` writes exactly one, Y != X,
    also at a point; no WCR, every access at depth 0;
  * ``g`` reads X only at constant offsets ``p + e`` (|e| <= 2) and ``f``
    does not read X.
"""

from __future__ import annotations

import os

from . import codegen as CG
from . import plan as P

# Off by default: measured 531 us per pair on heat_3d N=400 against 426 us
# for the two march-mode sweeps — the saved HBM pass is outweighed by the
# halo recomputation and L1 traffic (ncu: L1 77 %, issue 60 %, DRAM 34 %).
TEMPORAL = os.environ.get("B2_TEMPORAL", "0") == "1"
ZCHUNK = int(os.environ.get("B2_PAIR_Z", "32"))  # outer-dim planes per CTA
PAIR_V = int(os.environ.get("B2_PAIR_V", "2"))  # planes produced per barrier step


def _point_writes(pl, grp):
    """{container: point key} of the group's memory writes, or None."""
    out = {}
    for mem in grp.members:
        for (c, w, wcr, depth, pt) in pl.member_accesses(mem, grp.params):
            if not w:
                continue
            if pl.placement.get(c, "memory") == "reg":
                continue
            if wcr is not None or depth != 0 or pt is None:
                return None
            if c in out and out[c] != pt:
                return None
            out[c] = pt
    return out


def _offsets(pt, params):
    offs = []
    if len(pt) != len(params):
        return None
    for d, (c0, co) in enumerate(pt):
        if co != ((params[d], 1),):
            return None
        offs.append(c0)
    return tuple(offs)


def pair_info(pl, g1, g2):
    """(X, Y, o1, emin, emax) when g1 -> g2 can run as one paired kernel."""
    for g in (g1, g2):
        if not isinstance(g, P.MapGroup) or g.schedule != "parallel" or len(g.params) != 3:
            return None
        if g.idx in getattr(pl, "in_region", set()):
            return None
    r1 = [CG._const_range(pl, r) for r in g1.ranges]
    r2 = [CG._const_range(pl, r) for r in g2.ranges]
    if any(r is None or r[1] != 1 or r[2] < 1 for r in r1) or r1 != r2:
        return None
    w1, w2 = _point_writes(pl, g1), _point_writes(pl, g2)
    if not w1 or not w2 or len(w1) != 1 or len(w2) != 1:
        return None
    (X, pt1), = w1.items()
    (Y, pt2), = w2.items()
    if X == Y:
        return None
    o1 = _offsets(pt1, g1.params)
    if o1 is None or _offsets(pt2, g2.params) is None:
        return None
    offs = set()
    for mem in g1.members:
        for (c, w, wcr, depth, pt) in pl.member_accesses(mem, g1.params):
            if c == X and not w:
                return None  # f reads its own output
            if depth != 0:
                return None
    for mem in g2.members:
        for (c, w, wcr, depth, pt) in pl.member_accesses(mem, g2.params):
            if depth != 0:
                return None
            if c == X:
                if w or pt is None:
                    return None
                e = _offsets(pt, g2.params)
                if e is None or max(abs(x) for x in e) > 2:
                    return None
                offs.add(e)
    if not offs:
        return None
    emin = tuple(min(e[d] for e in offs) for d in range(3))
    emax = tuple(max(e[d] for e in offs) for d in range(3))
    return X, Y, o1, emin, emax


def find_pairs(pl) -> list:
    """Adjacent (g1, g2) map groups of every planned op sequence that pair."""
    out = []
    if not TEMPORAL:
        return out
    for head, ops in pl.ops.items():
        i = 0
        while i + 1 < len(ops):
            info = pair_info(pl, ops[i], ops[i + 1])
            if info is not None:
                out.append((ops[i], ops[i + 1]) + info)
                i += 2
            else:
                i += 1
    return out


def generate_pair(pl, g1, g2, X, Y, o1, emin, emax, shapes, name) -> CG.KernelSpec:
    gen1 = CG._Gen(pl, g1, shapes, name)
    gen2 = CG._Gen(pl, g2, shapes, name)
    spec = gen1.spec
    gen2.spec = spec
    gen2.uid = 100000
    gen1.place_override = {X: "reg"}
    gen2.ptr_override = {Y: "c_Yalt"}
    gen2.stencil = {X: {"min": emin, "max": emax}}
    # f at the ring point q (its own parameter names)
    env1 = {p: f"q_{i}" for i, p in enumerate(g1.params)}
    env2 = {p: f"p_{p}" for p in g2.params}
    for gen, grp, env in ((gen1, g1, env1), (gen2, g2, env2)):
        for mem in grp.members:
            for a in pl.member_accesses(mem, grp.params):
                if a[1]:
                    gen.written.add(a[0])
        gen.ind = 10 if gen is gen1 else 8
        start = len(gen.lines)
        for mem in grp.members:
            menv = {mp: env[gp] for mp, gp in mem.rename.items()}
            if mem.tasklet is not None:
                gen.tasklet(mem.state, mem.tasklet, menv, 0)
            else:
                gen.scope(mem.state, mem.entry, menv, 0)
        gen.body = gen.lines[start:]
    if spec.uses_flag:
        raise P.PlanError("guarded accesses in a paired sweep")
    yalt = gen1.arg(("ptr", Y + "#alt"))
    spec.containers = list(dict.fromkeys(spec.containers + [X, Y]))
    ct = CG.CT[pl.g.containers[X].dtype]
    cy = CG.CT[pl.g.containers[Y].dtype]
    rng = [CG._const_range(pl, r) for r in g1.ranges]
    SD = emax[0] - emin[0] + 1
    SY = 8 + emax[1] - emin[1]
    SX = 32 + emax[2] - emin[2]

    pro = [f'extern "C" __global__ void __launch_bounds__({SX * SY}) '
           f"{name}(const __grid_constant__ B2Args a) {{", "  B2_PDL_ENTRY();"]
    for c in spec.containers:
        if gen1.place(c) == "reg" and gen2.place(c) == "reg":
            continue
        if pl.placement.get(c, "memory") != "memory" and c != X:
            continue
        cd = pl.g.containers[c]
        q = "" if c == X else "const "
        pro.append(f"  {q}{CG.CT[cd.dtype]} *__restrict__ c_{c} = ({q}{CG.CT[cd.dtype]} *)"
                   f"{gen1.arg(('ptr', c))};")
        st = CG._row_major(shapes[c])
        for d in range(len(st)):
            pro.append(f"  constexpr b2_ll st_{c}_{d} = {st[d]}LL;")
        n = 1
        for x in shapes[c]:
            n *= x
        pro.append(f"  constexpr b2_ll sz_{c} = {n}LL;")
    pro.append(f"  {cy} *__restrict__ c_Yalt = ({cy} *){yalt};")
    for sname in spec.syms:
        if sname in pl.fixed:
            pro.append(f"  constexpr b2_ll s_{sname} = {int(pl.fixed[sname])}LL;")
        else:
            raise P.PlanError("loop-assigned symbol in a paired sweep")
    for i, (b, _, n) in enumerate(rng):
        pro.append(f"  constexpr b2_ll rb{i} = {b}LL, rl{i} = {n}LL;")
    for d in range(3):
        pro.append(f"  constexpr b2_ll o1_{d} = {o1[d]}LL, emin{d} = {emin[d]}LL, "
                   f"emax{d} = {emax[d]}LL;")
    xs = CG._row_major(shapes[X])
    V = PAIR_V
    BX, BY = SX, SY  # one thread per ring column (tile + halo)
    RS = 1
    while RS < SD + V - 1:
        RS *= 2  # power-of-two ring: slot arithmetic is a mask
    pro += [
        f"  constexpr int SDEPTH = {RS}, SY = {SY}, SX = {SX}, ZC = {ZCHUNK}, V = {V};",
        f"  __shared__ {ct} sm_{X}[SDEPTH][SY][SX];",
        "  constexpr b2_ll tiles_x = (rl2 + 31) / 32, tiles_y = (rl1 + 7) / 8;",
        "  constexpr b2_ll nch = (rl0 + ZC - 1) / ZC;",
        "  const b2_ll nvb = tiles_x * tiles_y * nch;",
        "  for (b2_ll vb = blockIdx.x; vb < nvb; vb += gridDim.x) {",
        "    const b2_ll tx = vb % tiles_x; b2_ll rem = vb / tiles_x;",
        "    const b2_ll ty = rem % tiles_y; const b2_ll tz = rem / tiles_y;",
        "    const b2_ll P1 = rb1 + ty * 8, P2 = rb2 + tx * 32;",
        "    const b2_ll zlo = rb0 + tz * ZC;",
        "    const b2_ll zhi = (zlo + ZC < rb0 + rl0 ? zlo + ZC : rb0 + rl0) - 1;",
        "    // this thread's ring column: X row yx, X column xx (fixed per tile)",
        "    const b2_ll yx = P1 + emin1 + threadIdx.y, xx = P2 + emin2 + threadIdx.x;",
        "    const b2_ll q_1 = yx - o1_1, q_2 = xx - o1_2;",
        "    const bool in12 = q_1 >= rb1 && q_1 < rb1 + rl1 && q_2 >= rb2 && q_2 < rb2 + rl2;",
        "    const bool own12 = q_1 >= P1 && q_1 < P1 + 8 && q_2 >= P2 && q_2 < P2 + 32;",
        f"    const bool inb12 = yx >= 0 && yx < {shapes[X][1]}LL && xx >= 0 && xx < {shapes[X][2]}LL;",
        "    const bool g2t = threadIdx.y < 8 && threadIdx.x < 32;",
        f"    const b2_ll p_{g2.params[1]} = P1 + threadIdx.y;",
        f"    const b2_ll p_{g2.params[2]} = P2 + threadIdx.x;",
        f"    const bool g2in = g2t && p_{g2.params[1]} < rb1 + rl1 && p_{g2.params[2]} < rb2 + rl2;",
        "    for (b2_ll zb = zlo + emin0; zb <= zhi + emax0; zb += V) {",
        "      // interior columns of full steps: branch-free unrolled planes, so",
        "      // the compiler reuses the outer-dim neighbours of f's loads",
        "      if (in12 && zb + V - 1 <= zhi + emax0 && zb - o1_0 >= rb0 &&",
        "          zb + V - 1 - o1_0 < rb0 + rl0) {",
        "#pragma unroll",
        "        for (int u = 0; u < V; ++u) {",
        "          const b2_ll zx = zb + u;",
        "          const b2_ll q_0 = zx - o1_0;",
        f"          const b2_ll xoff = zx * {xs[0]}LL + yx * {xs[1]}LL + xx * {xs[2]}LL;",
    ]
    regs1 = [c for c in spec.containers if gen1.place(c) == "reg"]
    loop = [f"          {CG.CT[pl.g.containers[c].dtype]} r_{c} = 0;" for c in regs1]
    loop += ["  " + ln for ln in gen1.body]
    loop += [
        f"          if (own12 && q_0 >= zlo && q_0 <= zhi) c_{X}[xoff] = r_{X};",
        f"          sm_{X}[(int)(zx - zlo - emin0) & (SDEPTH - 1)][threadIdx.y][threadIdx.x] = r_{X};",
        "        }",
        "      } else {",
        "#pragma unroll",
        "      for (int u = 0; u < V; ++u) {",
        "        const b2_ll zx = zb + u;",
        "        if (zx <= zhi + emax0) {",
        "          const b2_ll q_0 = zx - o1_0;",
        f"          const b2_ll xoff = zx * {xs[0]}LL + yx * {xs[1]}LL + xx * {xs[2]}LL;",
        f"          {ct} val;",
        "          if (in12 && q_0 >= rb0 && q_0 < rb0 + rl0) {",
    ]
    loop += [f"            {CG.CT[pl.g.containers[c].dtype]} r_{c} = 0;" for c in regs1]
    loop += ["    " + ln for ln in gen1.body]
    loop += [
        f"            val = r_{X};",
        f"            if (own12 && q_0 >= zlo && q_0 <= zhi) c_{X}[xoff] = val;",
        "          } else {",
        f"            val = (inb12 && zx >= 0 && zx < {shapes[X][0]}LL) ? c_{X}[xoff] : ({ct})0;",
        "          }",
        f"          sm_{X}[(int)(zx - zlo - emin0) & (SDEPTH - 1)][threadIdx.y][threadIdx.x] = val;",
        "        }",
        "      }",
        "      }",
        "      __syncthreads();",
        "#pragma unroll",
        "      for (int u = 0; u < V; ++u) {",
        "        const b2_ll pz = zb + u - emax0;",
        "        if (g2in && pz >= zlo && pz <= zhi) {",
        "          const int it = (int)(pz - zlo);",
        f"          const b2_ll p_{g2.params[0]} = pz;",
        "          const int v = 0;",
        "          (void)v; (void)it;",
    ]
    regs2 = [c for c in spec.containers if gen2.place(c) == "reg" and c != X]
    loop += [f"          {CG.CT[pl.g.containers[c].dtype]} r_{c} = 0;" for c in regs2]
    loop += ["  " + ln for ln in gen2.body]
    loop += ["        }", "      }", "      __syncthreads();", "    }", "  }", "}"]
    head = ["// paired stencil sweeps (temporal.py): "
            f"{g1.state.label} -> {g2.state.label}, ring of {SD} planes",
            "struct B2Args { long long w[%d]; };" % max(1, len(spec.args))]
    spec.source = "\n".join(head + pro + loop) + "\n"
    spec.mode = "pair"
    spec.block = (BX, BY, 1)
    spec.params = list(g2.params)
    spec.pair = (g1.idx, g2.idx, X, Y)
    spec.pair_geom = rng
    return spec


def pair_geometry(spec) -> tuple:
    rng = spec.pair_geom
    nvb = -(-rng[2][2] // 32) * -(-rng[1][2] // 8) * -(-rng[0][2] // ZCHUNK)
    return (max(1, min(nvb, CG.MAX_BLOCKS * 8)), 1, 1), spec.block
