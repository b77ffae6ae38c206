"""CPU tier: oracle pinned to the reference, IR/parsers, planner, NVRTC
compilation of every generated kernel, and the C ABI exports."""

import math
import re

import numpy as np
import pytest

from conftest import GOLDEN, MANIFEST, ROOT, golden_cases, load_case, rel_err


# --- the oracle restatement is pinned bitwise to the reference ------------------

@pytest.mark.parametrize("name,variant,case", golden_cases(1),
                         ids=lambda x: x if isinstance(x, str) else x.get("file", ""))
def test_oracle_restatement_matches_reference(name, variant, case):
    from oracle import interp_ref
    from paper_2107_00555_b200 import sdfg

    g = sdfg.load(GOLDEN / "graphs" / f"{name}.{variant}.json")
    d, inputs = load_case(case)
    c = interp_ref.Counters()
    out = interp_ref.interpret(g, case["symbols"], inputs, counters=c)
    key = f"interp_{variant}/"
    for k in [f[len(key):] for f in d.files if f.startswith(key)]:
        assert np.array_equal(out[k], d[key + k], equal_nan=True), f"{name}.{variant}:{k}"
    ref = case["counters"][variant]
    assert (c.map_iterations, c.wcr_commits) == (ref["map_iterations"], ref["wcr_commits"])
    if variant != "b2reg":
        # (b2reg: the reference interpreter also counts the wrapper's
        # copy-in / copy-out bytes, interp.py:491-517; the loader inlines it)
        assert c.bytes_moved == ref["bytes_moved"]


def test_reference_kats():
    """KATs of pkg/tests/test_interp.py:17-40, 122-139 against the oracle."""
    from oracle import interp_ref
    from paper_2107_00555_b200 import sdfg

    g = sdfg.load(GOLDEN / "graphs" / "jacobi_1d.raw.json")
    out = interp_ref.interpret(g, {"N": 4, "TSTEPS": 2},
                               {"A": np.array([0.0, 3.0, 0.0, 3.0]), "B": np.zeros(4)})
    assert np.array_equal(out["B"], [0.0, 0.99999, 1.99998, 0.0])
    g = sdfg.load(GOLDEN / "graphs" / "wcr_sum.raw.json")
    c = interp_ref.Counters()
    out = interp_ref.interpret(g, {"NI": 2, "NJ": 2}, {"alpha": 0.0, "C": np.ones((2, 2))},
                               counters=c)
    assert out["alpha"][()] == 4.0 and c.wcr_commits == 4
    g = sdfg.load(GOLDEN / "graphs" / "gemm.raw.json")
    A = np.array([[1.0, 2.0], [3.0, 4.0]])
    out = interp_ref.interpret(g, {"NI": 2, "NJ": 2, "NK": 2},
                               {"A": A, "B": np.eye(2), "C": np.zeros((2, 2)),
                                "alpha": 1.0, "beta": 0.0})
    assert np.array_equal(out["C"], A)
    g = sdfg.load(GOLDEN / "graphs" / "jacobi_2d.raw.json")
    out = interp_ref.interpret(g, {"N": 6, "TSTEPS": 2},
                               {"A": np.full((6, 6), 3.0), "B": np.full((6, 6), 3.0)})
    assert np.allclose(out["B"][1:-1, 1:-1], 3.0, rtol=0, atol=1e-14)


def test_reference_interp_equals_oracle_in_manifest():
    """Raw graphs interpret bitwise-equal to evaluate_program (reference
    criterion test_oracle_suite.py:47-48) — recorded at generation time."""
    for name, ent in MANIFEST["kernels"].items():
        for case in ent["cases"]:
            assert case["interp_equals_oracle"]["raw"], (name, case["file"])


# --- parsers and IR --------------------------------------------------------------

def test_symexpr():
    from paper_2107_00555_b200 import symexpr as S

    e = S.parse("(-4) * N + N * N + 4")
    assert S.evaluate(e, {"N": 10}) == 64
    assert S.evaluate(S.parse("-7 // 2"), {}) == -4
    assert S.evaluate(S.parse("min(N, 3) + max(1, M)"), {"N": 5, "M": 0}) == 4
    assert S.affine(S.parse("k0 + 1"), ("k0",), {}) == (1, {"k0": 1})
    assert S.affine(S.parse("2 * (i + N)"), ("i",), {"N": 3}) == (6, {"i": 2})
    assert S.affine(S.parse("i * j"), ("i", "j"), {}) is None
    assert S.interval(S.parse("i - 2 * j"), {"i": (0, 5), "j": (1, 3)}, {}) == (-6, 3)
    dims = S.parse_subset("1:N - 2:1, k0 + 1")
    assert [list(r) for r in S.eval_subset(dims, {"N": 5, "k0": 2})] == [[1, 2, 3], [3]]


def test_scalar_semantics_host():
    from paper_2107_00555_b200 import scalar as T

    assert T.evaluate(T.parse("i / NPT"), {"i": 3, "NPT": 4}) == 0.75
    assert T.evaluate(T.parse("-7.0 // 2.0"), {}) == -4.0
    assert T.evaluate(T.parse("(a < b) * c"), {"a": 1.0, "b": 2.0, "c": 5.0}) == 5.0
    assert math.isnan(T.evaluate(T.parse("min(x, 1.0)"), {"x": float("nan")}))
    assert T.evaluate(T.parse("min(1.0, x)"), {"x": float("nan")}) == 1.0
    assert T.evaluate(T.parse("c ? 1 : 2"), {"c": 0}) == 2
    code, ty = T.emit(T.parse("i / NPT <= in1 and in1 < 2"), {"i": "i", "NPT": "i", "in1": "f"})
    assert ty == "b" and "(double)" in code
    assert T.c_literal_f(0.2) == (0.2).hex()


def test_graph_loader_all_golden():
    from paper_2107_00555_b200 import sdfg

    for p in sorted((GOLDEN / "graphs").glob("*.json")):
        g = sdfg.load(p)
        for st in g.states:
            st.topological()
            st.scope_parents()
        assert g.start in {s.label for s in g.states}


def test_schema_errors():
    from paper_2107_00555_b200 import sdfg

    with pytest.raises(sdfg.SchemaError):
        sdfg.loads("{}")
    with pytest.raises(sdfg.SchemaError):
        sdfg.from_dict({"version": 2})
    with pytest.raises(sdfg.SchemaError):
        sdfg.loads("not json")


# --- planner and generated code ------------------------------------------------

def _modes(name, syms):
    from paper_2107_00555_b200 import codegen, plan as P, sdfg

    g = sdfg.load(GOLDEN / "graphs" / f"{name}.json")
    pl = P.Planner(g, syms).build()
    out = {}
    for op in pl.all_ops:
        if isinstance(op, P.MapGroup) and op.idx not in pl.in_region:
            out[op.idx] = codegen.generate(pl, op, pl.shapes(syms), f"k{op.idx}").mode
    regs = [codegen.generate_region(pl, r, pl.shapes(syms), "r") for r in pl.regions]
    return out, regs, pl


def test_kernel_mode_selection():
    """The schedules each benchmark program gets (DESIGN.md kernel families):
    heat_3d sweeps march along dim 0; softmax's exp+sum map is a warp-per-row
    reduction and its max loop a warp fold; the tiled-WCR conv2d (auto graph)
    accumulates in registers (thread-private stack accumulator in registers);
    go_fast's trace loop (pipe graph) is a register reduction."""
    m, _, _ = _modes("heat_3d.raw", {"N": 400, "TSTEPS": 100})
    assert set(m.values()) == {"march"}
    # march tiles are 64 x 8 and bulk-prefetch their input rows into L2
    from paper_2107_00555_b200 import codegen as CG, plan as P_, sdfg as S_
    syms_h = {"N": 400, "TSTEPS": 100}
    gh = S_.load(GOLDEN / "graphs" / "heat_3d.raw.json")
    plh = P_.Planner(gh, syms_h).build()
    grp = next(o for o in plh.all_ops if isinstance(o, P_.MapGroup))
    sp = CG.generate(plh, grp, plh.shapes(syms_h), "h")
    assert sp.block == (64, 8, 1) and "b2_prefetch_l2" in sp.source
    # opt-in tma3 (B2_TMA3=1): 60 x 16 tiles, one 62 x 18 x 1 f64 TMA box per
    # plane into a ring, producer warp + 8 consumer warps, 32-plane chunks
    CG.TMA3 = True
    try:
        sp = CG.generate(plh, grp, plh.shapes(syms_h), "h")
    finally:
        CG.TMA3 = False
    assert sp.mode == "tma3" and sp.block == (32, 9, 1) and sp.tmaps == [("A", (62, 18, 1))]
    assert "cp.async.bulk.tensor.3d" in sp.source and sp.grid_cap == 7 * 25 * 13
    m, regs, _ = _modes("softmax.raw", {"N": 64, "H": 16, "SM": 512})
    assert "rowred" in m.values()
    assert len(regs) == 1 and regs[0].warp
    m, _, _ = _modes("conv2d_bias.auto", {"NB": 8, "H": 256, "W": 256, "CI": 3, "CO": 16,
                                          "K": 20, "HO": 237, "WO": 237})
    assert "reduce" in m.values()
    # raw conv2d: the 7-D WCR map is a contraction out[m, c] += inp[m, k] *
    # w[k, c] -> implicit GEMM on DMMA (M = 8*237*237, N = 16, K = 20*20*3);
    # with the contraction mode off, the output channel is register-blocked
    from paper_2107_00555_b200 import codegen, plan as P, sdfg
    syms = {"NB": 8, "H": 256, "W": 256, "CI": 3, "CO": 16, "K": 20, "HO": 237, "WO": 237}
    g = sdfg.load(GOLDEN / "graphs" / "conv2d_bias.raw.json")
    pl = P.Planner(g, syms).build()
    grp = [op for op in pl.all_ops if isinstance(op, P.MapGroup)][1]
    sp = codegen.generate(pl, grp, pl.shapes(syms), "k1")
    # inp[n, i + ki, j + kj, ci] slides along j (stride 3) and (kj, ci) is a
    # contiguous run of 60 addresses: one 825-double window per (tile, ki)
    assert sp.mode == "contract" and sp.contract == {
        "M": 449352, "N": 16, "K": 1200, "TN": 16, "TM": 256, "tiles_m": 8 * 237,
        "slide": {"S": 3, "BK": 60, "KR": 60, "WS": 826, "jm": "j"}}
    assert "sliding-window contraction" in sp.source
    assert "mma.sync.aligned.m16n8k4.row.col.f64" in sp.source
    codegen.CONTRACT_SLIDE = False
    try:
        sp = codegen.generate(pl, grp, pl.shapes(syms), "k1")
    finally:
        codegen.CONTRACT_SLIDE = True
    assert sp.mode == "contract" and sp.contract == {"M": 449352, "N": 16, "K": 1200, "TN": 16,
                                                     "TM": 256}
    assert sp.smem > 48 * 1024  # dynamic shared memory (two 256 x 20 A stages)
    # a plain GEMM has no sliding operand (A's row stride is K)
    gm = sdfg.load(GOLDEN / "graphs" / "matmul.auto.json")
    msy = {"M": 4096, "K": 4096, "N": 4096}
    plm = P.Planner(gm, msy).build()
    specs = [codegen.generate(plm, op, plm.shapes(msy), f"k{op.idx}") for op in plm.all_ops
             if isinstance(op, P.MapGroup) and op.schedule == "parallel"]
    assert any(x.mode == "contract" and "slide" not in x.contract for x in specs)
    codegen.CONTRACT_MODE = False
    try:
        sp = codegen.generate(pl, grp, pl.shapes(syms), "k1")
    finally:
        codegen.CONTRACT_MODE = True
    assert sp.mode == "reduce" and "_v[16]" in sp.source and "NOUTB = 449352LL" in sp.source
    m, _, _ = _modes("go_fast.pipe", {"N": 12000})
    assert "reduce" in m.values()


def test_rowpass_tma_selection():
    """atax / bicg rows stream through the TMA bulk-copy ring; gemver's
    prologue pass keeps the register-prefetch kernel; odd row pitches (not
    16-byte multiples) fall back too."""
    from paper_2107_00555_b200 import plan as P, sdfg

    def rowpasses(name, syms):
        g = sdfg.load(GOLDEN / "graphs" / f"{name}.json")
        pl = P.Planner(g, syms).build()
        out = []
        for op in pl.all_ops:
            rp = getattr(op, "rowpass", None)
            if rp is not None:
                rp.source(pl.shapes(syms), f"t{op.idx}")
                out.append(rp)
        return out

    assert all(rp.tma for rp in rowpasses("atax.raw", {"M": 8000, "N": 8000}))
    assert all(rp.tma for rp in rowpasses("bicg.raw", {"N": 8000, "M": 8000}))
    gv = rowpasses("gemver.raw", {"N": 8000})
    assert any(not rp.tma for rp in gv)
    assert not any(rp.tma for rp in rowpasses("atax.raw", {"M": 3000, "N": 2501}))


def test_fusion_collapses_heat3d_chain():
    """heat_3d's ~16 maps per sweep (reference subgraph_fusion crashes on it,
    SURVEY.md §0) fuse into one kernel per half-sweep with every
    intermediate in registers."""
    from paper_2107_00555_b200 import plan as P, sdfg

    g = sdfg.load(GOLDEN / "graphs" / "heat_3d.raw.json")
    pl = P.Planner(g, {"N": 400, "TSTEPS": 100}).build()
    maps = [op for op in pl.all_ops if isinstance(op, P.MapGroup)]
    assert len(maps) == 2
    assert all(len(m.members) >= 15 for m in maps), [len(m.members) for m in maps]
    temps = [n for n, c in g.containers.items() if c.transient]
    assert all(pl.placement[t] == "reg" for t in temps)


def test_jacobi_stencil_not_fused_across_sweeps():
    from paper_2107_00555_b200 import plan as P, sdfg

    g = sdfg.load(GOLDEN / "graphs" / "jacobi_2d.raw.json")
    pl = P.Planner(g, {"N": 2000, "TSTEPS": 100}).build()
    maps = [op for op in pl.all_ops if isinstance(op, P.MapGroup)]
    assert len(maps) == 2  # B-sweep and A-sweep need a global barrier


def test_all_generated_kernels_compile_for_sm100a():
    """Every kernel the planner generates for every golden graph compiles
    with NVRTC for sm_100a (no GPU needed)."""
    from paper_2107_00555_b200 import codegen, plan as P, runtime as rt, sdfg

    rt.load_library()
    n = 0
    for name, ent in MANIFEST["kernels"].items():
        for v in ent["variants"]:
            g = sdfg.load(GOLDEN / "graphs" / f"{name}.{v}.json")
            pl = P.Planner(g, ent["cases"][-1]["symbols"]).build()
            for op in pl.all_ops:
                if isinstance(op, P.MapGroup):
                    spec = codegen.generate(pl, op, pl.shapes(ent["cases"][-1]["symbols"]), f"b2_map_{g.name}_{op.idx}")
                    cub, _ = rt.get_cubin(rt.family_source("prelude.cuh") + "\n" + spec.source,
                                          spec.name)
                    assert len(cub) > 0
                    n += 1
    assert n > 50


# --- C ABI -----------------------------------------------------------------------

def test_libb2_exports_every_declared_symbol():
    from paper_2107_00555_b200 import runtime as rt

    header = (ROOT / "include" / "b2.h").read_text()
    declared = set(re.findall(r"\b(b2_\w+)\s*\(", header))
    lib = rt.load_library()
    for sym in sorted(declared):
        assert hasattr(lib, sym), f"libb2.so does not export {sym}"
    assert declared == set(rt.EXPORTS)
    assert lib.b2_version() == 1


def test_no_gpu_fails_loudly():
    """Without a device the backend raises instead of falling back to CPU."""
    from paper_2107_00555_b200 import runtime as rt

    n = __import__("ctypes").c_int(0)
    rt.lib().b2_device_count(__import__("ctypes").byref(n))
    if n.value > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(rt.BackendUnavailable):
        rt.device(0)


def test_rowpass_fusions_plan_and_compile():
    """gemver / atax / bicg fold their MATMUL nodes (and gemver's A-update
    map) into single rowpass passes that compile for sm_100a."""
    from paper_2107_00555_b200 import plan as P, runtime as rt, sdfg

    rt.load_library()
    want = {"gemver.raw": ["axpy+pro", "dot"], "atax.raw": ["dot,axpy+coefdot"],
            "bicg.raw": ["axpy,dot"]}
    for name, kinds in want.items():
        g = sdfg.load(GOLDEN / "graphs" / f"{name}.json")
        syms = {"gemver.raw": {"N": 8000}, "atax.raw": {"M": 8000, "N": 8000},
                "bicg.raw": {"N": 8000, "M": 8000}}[name]
        pl = P.Planner(g, syms).build()
        got = []
        for op in pl.all_ops:
            if isinstance(op, P.LibOp) and op.rowpass is not None:
                rp = op.rowpass
                got.append(",".join(m.kind for m in rp.mvs) + ("+pro" if rp.prologue else "")
                           + ("+coefdot" if rp.coef_from_dot else ""))
                src = rp.source(pl.shapes(), f"{g.name}_{op.idx}")
                assert rt.get_cubin(src, f"b2_rp_{g.name}_{op.idx}")[0]
        assert got == kinds, (name, got)


def test_init_fill_fusion_detected():
    """machine._init_fusions: nbody's nested get_acc graph pairs its
    constant fill (acc[:] = 0.0) with the following pair-force reduction,
    whose targets acc[i, 0..2] cover the whole container."""
    from paper_2107_00555_b200 import machine, plan as P, sdfg

    g = sdfg.load(GOLDEN / "graphs" / "nbody.raw.json")
    pl = P.Planner(g, {"N": 100, "NT": 10}).build()
    nested = [o for o in pl.all_ops if isinstance(o, P.NestedOp)][0]
    pl2 = P.Planner(nested.node.sdfg, {"N": 100}).build()

    class _Ex:
        pass

    ex = _Ex()
    ex.planner, ex.buf, ex.init_skip = pl2, _Ex(), set()
    ex.buf.shape = pl2.shapes({"N": 100})
    ex._const_fill = machine.GpuExecutor._const_fill.__get__(ex)
    fused = machine.GpuExecutor._init_fusions(ex)
    assert fused == {1: {"acc": "0.0"}} and ex.init_skip == {0}


@pytest.mark.parametrize("name,syms,cont,expect", [
    ("softmax.raw", {"N": 2, "H": 3, "SM": 64}, "ex", True),     # point write, same-point re-read
    ("atax.raw", {"M": 30, "N": 20}, "tmp0", True),               # full MATMUL output
    ("softmax.raw", {"N": 2, "H": 3, "SM": 64}, "sm", False),     # WCR target: needs its zeros
])
def test_transient_overwrite_analysis(name, syms, cont, expect):
    """machine.GpuExecutor._overwrites: a scope transient whose first op
    writes every element before any read is not zeroed per call."""
    from paper_2107_00555_b200 import machine, plan as P, sdfg

    g = sdfg.load(GOLDEN / "graphs" / f"{name}.json")
    pl = P.Planner(g, syms).build()

    class _Ex:
        pass

    ex = _Ex()
    ex.planner, ex.buf, ex.bindings = pl, _Ex(), dict(syms)
    ex.buf.shape = pl.shapes(syms)
    first = next(op for op in pl.all_ops
                 if cont in pl.op_reads.get(op.idx, set()) | pl.op_writes.get(op.idx, set()))
    assert machine.GpuExecutor._overwrites(ex, cont, first) is expect


@pytest.mark.parametrize("name,syms,expect", [
    # mx is touched by a device loop region (the max nest): never skipped;
    # ex is written point-wise then re-read at the same point: skipped;
    # sm is a WCR target that needs its zeros
    ("softmax.raw", {"N": 2, "H": 3, "SM": 64}, {"ex"}),
    # nbody: tmp0..2 (vel/pos update temporaries) are written point-wise
    # over their whole [0:N-1, 0:2] box before any read: skipped
    ("nbody.raw", {"N": 9, "NT": 2}, {"tmp0", "tmp1", "tmp2"}),
])
def test_zero_skip_set_from_dry_run(name, syms, expect):
    """run the real dry-run analysis (_dead_on_entry) and pin the
    exact zero-skip set, so region-touched containers stay zeroed."""
    from paper_2107_00555_b200 import machine, plan as P, sdfg

    g = sdfg.load(GOLDEN / "graphs" / f"{name}.json")
    ex = object.__new__(machine.GpuExecutor)
    ex.g, ex.bindings = g, dict(syms)
    ex.opt = machine.InterpOptions()
    ex.planner = P.Planner(g, ex.bindings).build()
    ex.planner.dynamic_p0 = False
    ex.comm, ex.capturable, ex.device_branching = None, True, False
    ex.buf = machine._Buffers()
    ex.buf.shape = ex.planner.shapes(syms)
    ex._exec_nested = lambda op, sym, counters, dry=False: None
    ex.pairs, ex.waves, ex._wave_elig, ex._wave_pending = {}, {}, {}, []
    ex.init_skip, ex.specs = set(), {}
    ex._dead_on_entry()
    assert ex.zero_skip == expect
    assert "mx" not in ex.zero_skip


def test_block_region_selection():
    """Loop nests whose inner loops iterate small maps (adi: TSTEPS x 4 j
    loops of one (N - 2)-point map each) become ONE single-CTA kernel; a
    stencil's time loop around its full-width maps stays host-driven (one
    kernel per map in the captured graph), and softmax's parallel row loops
    keep their warp-fold region."""
    from paper_2107_00555_b200 import codegen, plan as P, sdfg

    def regions(name, syms):
        g = sdfg.load(GOLDEN / "graphs" / f"{name}.json")
        pl = P.Planner(g, syms).build()
        return pl, [(r.loop.var, r.block, [l.var for l in r.par]) for r in pl.regions]

    for v in ("raw", "pipe", "auto"):
        pl, regs = regions(f"adi.{v}", {"N": 400, "TSTEPS": 5})
        assert regs == [("t", True, [])], (v, regs)
        spec = codegen.generate_region(pl, pl.regions[0], pl.shapes({"N": 400, "TSTEPS": 5}), "r")
        assert spec.block_region and spec.block == (416, 1, 1)
        assert "__syncthreads();" in spec.source and "if (blockIdx.x != 0) return;" in spec.source
    assert regions("jacobi_2d.raw", {"N": 34, "TSTEPS": 5})[1] == []
    assert regions("heat_3d.raw", {"N": 12, "TSTEPS": 3})[1] == []
    assert regions("softmax.raw", {"N": 1, "H": 2, "SM": 40})[1] == [("i", False, ["i", "j", "k"])]
    # maps larger than one CTA sweeps per step stay full-width kernels
    assert regions("adi.pipe", {"N": 5000, "TSTEPS": 2})[1] == []


def test_rowred_prefetches_next_row():
    """softmax's exp+sum row reduction: lane 0 L2-prefetches the warp's next
    row of x (the only read-only input walked along the row); the per-row
    maximum mx is not prefetched (no row-parameter dimension)."""
    from paper_2107_00555_b200 import codegen as CG, plan as P_, sdfg as S_

    syms = {"N": 2, "H": 2, "SM": 512}
    g = S_.load(GOLDEN / "graphs" / "softmax.raw.json")
    pl = P_.Planner(g, syms).build()
    specs = [CG.generate(pl, o, pl.shapes(syms), f"s{o.idx}") for o in pl.all_ops
             if isinstance(o, P_.MapGroup)]
    rr = [sp for sp in specs if sp.mode == "rowred"]
    assert rr and CG.ROWRED_PF
    src = rr[0].source
    assert "const b2_ll rown = row + " in src
    assert src.count("b2_prefetch_l2(") == 1 and "c_x + e0" in src.replace("(const char *)", "")
