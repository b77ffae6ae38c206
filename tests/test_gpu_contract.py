"""The reference interpreter's own contract tests (pkg/tests/test_interp.py),
run against the B200 executor on graphs the reference compiled (golden
graphs; the extra programs come from tests/golden/make_extra_graphs.py)."""

import numpy as np
import pytest

from conftest import GOLDEN, rel_err

pytestmark = pytest.mark.gpu


def _g(name):
    from paper_2107_00555_b200 import sdfg

    return sdfg.load(GOLDEN / "graphs" / f"{name}.json")


def _ctx(bindings, inputs):
    from paper_2107_00555_b200 import ExecContext

    return ExecContext(bindings=dict(bindings)).bind_inputs(inputs)


def test_gemm_identity():
    """test_interp.py:17-24"""
    from paper_2107_00555_b200 import interpret

    A = np.array([[1.0, 2.0], [3.0, 4.0]])
    out = interpret(_g("gemm.raw"), _ctx({"NI": 2, "NJ": 2, "NK": 2},
                                         {"A": A, "B": np.eye(2), "C": np.zeros((2, 2)),
                                          "alpha": 1.0, "beta": 0.0}))
    assert np.array_equal(out["C"], A)


def test_jacobi_first_half_step():
    """test_interp.py:26-32: the inexact 0.33333 coefficient, bitwise."""
    from paper_2107_00555_b200 import interpret

    out = interpret(_g("jacobi_1d.raw"), _ctx({"N": 4, "TSTEPS": 2},
                                              {"A": np.array([0.0, 3.0, 0.0, 3.0]),
                                               "B": np.zeros(4)}))
    assert np.array_equal(out["B"], [0.0, 0.99999, 1.99998, 0.0])


def test_wcr_sum_of_ones():
    """test_interp.py:34-40: value and commit count."""
    from paper_2107_00555_b200 import interpret

    ctx = _ctx({"NI": 2, "NJ": 2}, {"alpha": 0.0, "C": np.ones((2, 2))})
    out = interpret(_g("wcr_sum.raw"), ctx)
    assert out["alpha"][()] == 4.0
    assert ctx.counters.wcr_commits == 4


@pytest.mark.parametrize("name,syms", [("gemm", {"NI": 4, "NJ": 6, "NK": 8}),
                                       ("jacobi_2d", {"N": 6, "TSTEPS": 4})])
def test_run_twice(name, syms):
    """test_interp.py:44-50"""
    from paper_2107_00555_b200 import run_twice_determinism
    from paper_2107_00555_b200 import symexpr

    g = _g(f"{name}.raw")
    rng = np.random.default_rng(3)
    inputs = {}
    for n, c in g.containers.items():
        if not c.transient:
            shape = tuple(symexpr.evaluate(d, syms) for d in c.shape)
            inputs[n] = rng.uniform(-1, 1, shape) if shape else float(rng.uniform(0.5, 1.5))
    assert run_twice_determinism(g, _ctx(syms, inputs))


def test_tiled_reduction_deterministic():
    """test_interp.py:52-64: tile_wcr(16) reduction, run twice bitwise; and
    the sum itself."""
    from paper_2107_00555_b200 import interpret, run_twice_determinism

    g = _g("tiled_red.raw")
    assert run_twice_determinism(g, _ctx({"N": 64}, {"s": 0.0, "A": np.arange(64.0)}))
    out = interpret(g, _ctx({"N": 64}, {"s": 0.0, "A": np.arange(64.0)}))
    assert out["s"][()] == 2016.0


def test_missing_binding():
    """test_interp.py:66-70"""
    from paper_2107_00555_b200 import interpret

    with pytest.raises(Exception, match="missing symbol"):
        interpret(_g("gemm.raw"), _ctx({"NI": 2, "NJ": 2}, {}))


def test_out_of_bounds_is_hard_error():
    """test_interp.py:72-81: the message carries the offending index."""
    from paper_2107_00555_b200 import OutOfBoundsError, interpret

    with pytest.raises(OutOfBoundsError) as exc:
        interpret(_g("oob_read.raw"), _ctx({"N": 4, "K": 9},
                                           {"A": np.zeros(4), "B": np.zeros(4)}))
    assert "9" in str(exc.value)


def test_shape_mismatch_rejected():
    """test_interp.py:83-90"""
    from paper_2107_00555_b200 import interpret

    with pytest.raises(Exception, match="shape"):
        interpret(_g("gemm.raw"), _ctx({"NI": 2, "NJ": 2, "NK": 2},
                                       {"A": np.zeros((3, 3)), "B": np.eye(2),
                                        "C": np.zeros((2, 2)), "alpha": 1.0, "beta": 0.0}))


def test_bytes_additive_over_states():
    """test_interp.py:93-112: splitting bicg into its two statements moves
    the same bytes in total."""
    from paper_2107_00555_b200 import interpret

    syms = {"N": 6, "M": 4}
    rng = np.random.default_rng(3)
    inputs = {"A": rng.uniform(-1, 1, (6, 4)), "s": rng.uniform(-1, 1, 4),
              "q": rng.uniform(-1, 1, 6), "p": rng.uniform(-1, 1, 4), "r": rng.uniform(-1, 1, 6)}
    ctx = _ctx(syms, {k: v.copy() for k, v in inputs.items()})
    interpret(_g("bicg.raw"), ctx)
    total = ctx.counters.bytes_moved
    assert total > 0
    parts = 0
    for piece in ("bicg_head.raw", "bicg_tail.raw"):
        cp = _ctx(syms, {k: v.copy() for k, v in inputs.items()})
        interpret(_g(piece), cp)
        parts += cp.counters.bytes_moved
    assert parts == total


def test_map_iterations_counted():
    """test_interp.py:114-121"""
    from paper_2107_00555_b200 import interpret

    ctx = _ctx({"NI": 3, "NJ": 5}, {"alpha": 0.0, "C": np.ones((3, 5))})
    interpret(_g("wcr_sum.raw"), ctx)
    assert ctx.counters.map_iterations == 15


def test_jacobi_1d_constant_field():
    """test_interp.py:123-130"""
    from paper_2107_00555_b200 import interpret

    c = 2.0
    out = interpret(_g("jacobi_1d.raw"), _ctx({"N": 6, "TSTEPS": 2},
                                              {"A": np.full(6, c), "B": np.full(6, c)}))
    assert np.allclose(out["B"][1:-1], 0.99999 * c, rtol=0, atol=1e-14)


def test_jacobi_2d_constant_field():
    """test_interp.py:132-140: the 0.2 coefficient is exact."""
    from paper_2107_00555_b200 import interpret

    c = 3.0
    out = interpret(_g("jacobi_2d.raw"), _ctx({"N": 6, "TSTEPS": 2},
                                              {"A": np.full((6, 6), c), "B": np.full((6, 6), c)}))
    assert np.allclose(out["B"][1:-1, 1:-1], c, rtol=0, atol=1e-14)


@pytest.mark.parametrize("s0", [2.5, -1.0, 0.0])
def test_condition_on_scalar_container(s0):
    """Transitions whose condition reads a 0-d container updated inside the
    loop (interp.py:265-274): evaluated on the host after a device sync."""
    from paper_2107_00555_b200 import interpret

    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, 37)
    out = interpret(_g("branchy.raw"), _ctx({"N": 37, "TSTEPS": 6}, {"x": x.copy(), "s": s0}))
    xr, s = x.copy(), s0
    for _ in range(6):
        if s > 0.0:
            xr = xr * 0.5
            s = s - 1.0
        else:
            xr = xr + 1.0
    assert np.array_equal(out["x"], xr) and out["s"][()] == s


@pytest.mark.parametrize("s0", [2.5, -1.0, 4.0])
def test_device_branches_match_host_branches(monkeypatch, s0):
    """The container-dependent branch captured as a CUDA conditional IF/ELSE
    node gives the same outputs and counters as host-evaluated conditions,
    across repeated graph replays with different inputs."""
    from paper_2107_00555_b200 import machine

    g = _g("branchy.raw")
    rng = np.random.default_rng(6)
    x = rng.uniform(-1, 1, 37)
    res = {}
    for mode in (True, False):
        monkeypatch.setattr(machine, "DEVICE_BRANCHES", mode)
        ex = machine.GpuExecutor(g, {"N": 37, "TSTEPS": 7})
        outs = []
        for s_in in (s0, -s0):
            keep = ex.prepare_inputs({"x": x.copy(), "s": s_in})
            c = machine.Counters()
            ex.run_device(first_call=True, counters=c)
            outs.append((ex.download("x"), ex.download("s"), c.as_dict()))
            ex.sync()
            del keep
        res[mode] = outs
        if mode:
            assert ex.device_branching and ex.graph_exec is not None
        ex.close()
    for (xa, sa, ca), (xb, sb, cb) in zip(res[True], res[False]):
        assert np.array_equal(xa, xb) and sa == sb
        assert ca == cb


def _azimint_inputs(seed, syms):
    from paper_2107_00555_b200 import symexpr

    g = _g("azimint_naive.auto")
    rng = np.random.default_rng(seed)
    out = {}
    for n, c in g.containers.items():
        if not c.transient:
            shape = tuple(symexpr.evaluate(d, syms) for d in c.shape)
            out[n] = rng.uniform(-1, 1, shape) if shape else float(rng.uniform(0.5, 1.5))
    return out


def test_persistent_transients_per_context():
    """PERSISTENT transients belong to ctx.persistent
    (interp.py:216-219).  Two fresh contexts on the SAME Graph object each
    start from zeros; azimint_naive.auto's acc/cnt take only WCR-add writes,
    so stale values would show."""
    from oracle import interp_ref
    from paper_2107_00555_b200 import interpret

    g = _g("azimint_naive.auto")
    syms = {"N": 301, "NPT": 7}
    for seed in (0, 1):
        inputs = _azimint_inputs(seed, syms)
        ref = interp_ref.interpret(g, syms, {k: np.array(v) for k, v in inputs.items()})
        ctx = _ctx(syms, inputs)
        out = interpret(g, ctx)
        for k in ref:
            assert np.allclose(out[k], ref[k], rtol=1e-12, atol=1e-12, equal_nan=True), (seed, k)
        assert set(ctx.persistent) == {"acc", "cnt"}


def test_persistent_transients_kept_in_same_context():
    """The same context twice: the second run starts from the persistent
    values the first left in ctx.persistent (the reference's semantics),
    and ctx.persistent holds the oracle's persistent arrays."""
    from oracle import interp_ref
    from paper_2107_00555_b200 import interpret

    g = _g("azimint_naive.auto")
    syms = {"N": 301, "NPT": 7}
    inputs = _azimint_inputs(5, syms)
    pers = {}
    interp_ref.interpret(g, syms, {k: np.array(v) for k, v in inputs.items()}, persistent=pers)
    ref = interp_ref.interpret(g, syms, {k: np.array(v) for k, v in inputs.items()},
                               persistent=pers)
    ctx = _ctx(syms, inputs)
    interpret(g, ctx)
    out = interpret(g, ctx)
    for k in ref:
        assert np.allclose(out[k], ref[k], rtol=1e-12, atol=1e-12, equal_nan=True), k
    for k in ("acc", "cnt"):
        assert np.allclose(ctx.persistent[k], pers[k], rtol=1e-12, atol=1e-12), k


def test_options_are_part_of_executor_key():
    from paper_2107_00555_b200 import InterpOptions
    from paper_2107_00555_b200.machine import get_executor

    g = _g("gemm.raw")
    b = {"NI": 4, "NJ": 6, "NK": 8}
    e1 = get_executor(g, b, InterpOptions())
    e2 = get_executor(g, b, InterpOptions(skip_validation=True))
    e3 = get_executor(g, b, InterpOptions(max_transitions=5))
    assert e1 is get_executor(g, b, None)
    assert len({id(e1), id(e2), id(e3)}) == 3


def test_skip_validation_runs_racy_graph():
    """With skip_validation the reference executes the racy graph (both
    unordered writes store x into all of A); so do we."""
    import json

    from paper_2107_00555_b200 import InterpOptions, interpret

    g = json.loads((GOLDEN / "validation_cases.json").read_text())["race_whole"]["graph"]
    out = interpret(g, _ctx({"N": 8}, {"A": np.zeros(8), "x": 2.5}),
                    InterpOptions(skip_validation=True))
    assert np.array_equal(out["A"], np.full(8, 2.5))


@pytest.mark.parametrize("name,syms", [("matmul.auto", {"M": 300, "K": 200, "N": 250}),
                                       ("matmul.auto", {"M": 257, "K": 129, "N": 130}),
                                       ("gemm.auto", {"NI": 190, "NJ": 220, "NK": 240})])
def test_blocked_matmul_expansion_runs_as_contraction(name, syms):
    """The reference's blocked MATMUL expansion (auto_optimize,
    autoopt.py:707-813: tile map around a sequential (i, j, k) map) is
    recognised as a contraction and runs on DMMA: equal to the reference
    interpreter's result within the tensor-core tolerance."""
    from oracle import interp_ref
    from paper_2107_00555_b200 import ExecContext, interpret, sdfg
    from paper_2107_00555_b200.machine import GpuExecutor

    g = sdfg.load(GOLDEN / "graphs" / f"{name}.json")
    ex = GpuExecutor(g, syms)
    try:
        assert any(sp.mode == "contract" for sp in ex.specs.values())
    finally:
        ex.close()
    rng = np.random.default_rng(sum(syms.values()))
    ins = {}
    for n, c in g.containers.items():
        if not c.transient:
            shp = tuple(sdfg.symexpr.evaluate(d, syms) for d in c.shape)
            ins[n] = rng.uniform(-1, 1, shp) if shp else np.float64(rng.uniform(0.5, 1.5))
    out = interpret(g, ExecContext(bindings=dict(syms)).bind_inputs({k: np.array(v) for k, v in ins.items()}))
    # the reference semantics in closed form (evaluate_program: BLAS matmul);
    # the blocked map's per-point Python reference would take minutes here
    if name.startswith("matmul"):
        ref = {"C": ins["A"] @ ins["B"]}
    else:
        ref = {"C": ins["alpha"] * ins["A"] @ ins["B"] + ins["beta"] * ins["C"]}
    for k in ref:
        assert rel_err(out[k], ref[k]) <= 1e-12, (k, rel_err(out[k], ref[k]))
    _ = interp_ref


@pytest.mark.parametrize("NB,H,W,K,BK", [(2, 30, 40, 8, 24), (2, 24, 300, 20, 60),
                                         (1, 40, 256, 20, 60), (2, 30, 60, 6, None)])
def test_sliding_window_contraction(NB, H, W, K, BK):
    """conv2d_bias's X operand slides along the output column (stride CI)
    with (kj, ci) a contiguous run of K * CI addresses: the contraction
    stages one window per (tile, k chunk) (BK = 24 for K = 8, 60 for K = 20;
    W = 300 gives two column tiles per output row, the second with idle
    m16 fragments; K = 6's run of 18 has no k-chunk divisor, so the generic
    gather runs).  Equal to the closed form within the tensor-core
    tolerance."""
    from paper_2107_00555_b200 import ExecContext, interpret, sdfg
    from paper_2107_00555_b200.machine import GpuExecutor

    CI, CO = 3, 16
    HO, WO = H - K + 1, W - K + 1
    syms = dict(NB=NB, H=H, W=W, CI=CI, CO=CO, K=K, HO=HO, WO=WO)
    g = sdfg.load(GOLDEN / "graphs" / "conv2d_bias.raw.json")
    ex = GpuExecutor(g, syms)
    try:
        slides = [sp.contract.get("slide") for sp in ex.specs.values() if sp.mode == "contract"]
    finally:
        ex.close()
    assert slides and (slides[0] or {}).get("BK") == BK
    rng = np.random.default_rng(K * W)
    inp = rng.uniform(-1, 1, (NB, H, W, CI))
    w = rng.uniform(-1, 1, (K, K, CI, CO))
    b = rng.uniform(-1, 1, CO)
    out = interpret(g, ExecContext(bindings=syms).bind_inputs(
        {"inp": inp, "w": w, "bias": b, "out": np.zeros((NB, HO, WO, CO))}))["out"]
    ref = np.broadcast_to(b, (NB, HO, WO, CO)).copy()
    for ki in range(K):
        for kj in range(K):
            ref += np.einsum("nijc,cd->nijd", inp[:, ki:ki + HO, kj:kj + WO, :], w[ki, kj])
    assert rel_err(out, ref) <= 1e-12, rel_err(out, ref)


def test_privatised_map_region_doitgen_raw(monkeypatch):
    """doitgen.raw's loops r, q, p around a map into the transient tmp0 and
    a REDUCE of tmp0 run as ONE thread-per-(r, q, p) region with tmp0
    private per thread (loops._map_regions): the same counters as the
    host-driven launch sequence, results within the f64 tolerance of it and
    of the closed form (the in-thread REDUCE sums sequentially, the library
    REDUCE in its own order)."""
    from paper_2107_00555_b200 import ExecContext, interpret, loops, sdfg
    from paper_2107_00555_b200.machine import GpuExecutor

    syms = {"NR": 8, "NQ": 8, "NP": 160}
    g = sdfg.load(GOLDEN / "graphs" / "doitgen.raw.json")
    ex = GpuExecutor(g, syms)
    try:
        regs = [(r.block, [l.var for l in r.par], sorted(r.private)) for r in ex.planner.regions]
    finally:
        ex.close()
    assert regs == [(False, ["r", "q", "p"], ["tmp0"])]
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (8, 8, 160))
    C4 = rng.uniform(-1, 1, (160, 160))

    def run(graph):
        ctx = ExecContext(bindings=dict(syms)).bind_inputs(
            {"A": A.copy(), "C4": C4.copy(), "out": np.zeros((8, 8, 160))})
        return interpret(graph, ctx), ctx.counters

    out, cnt = run(g)
    monkeypatch.setattr(loops, "MAP_REGIONS", False)
    g2 = sdfg.load(GOLDEN / "graphs" / "doitgen.raw.json")
    out2, cnt2 = run(g2)
    ref = np.einsum("rqs,sp->rqp", A, C4)
    assert rel_err(out["out"], ref) <= 1e-12
    assert rel_err(out["out"], out2["out"]) <= 1e-12
    assert (cnt.map_iterations, cnt.wcr_commits) == (cnt2.map_iterations, cnt2.wcr_commits)
    assert cnt.map_iterations == 8 * 8 * 160 * 160


@pytest.mark.parametrize("variant,NP", [("pipe", 256), ("b2reg", 256), ("auto", 256), ("auto", 250)])
def test_map_reduce_contraction_doitgen(variant, NP):
    """doitgen's LoopToMap form — a map over (r, q, p) whose scope maps
    T[k] = A[r, q, k] * C4[k, p] into a transient row and REDUCEs it into
    out[r, q, p] — runs as the DMMA contraction with zero-initialised
    accumulators (T never materialised): within the tensor-core tolerance
    of the closed form.  The auto form (auto_optimize's tiled REDUCE: O = 0,
    per 16-wide tile acc += T[k], O += acc) is the same sum; NP = 250 leaves
    a partial last tile."""
    from paper_2107_00555_b200 import ExecContext, interpret, sdfg
    from paper_2107_00555_b200.machine import GpuExecutor

    syms = {"NR": 8, "NQ": 12, "NP": NP}
    g = sdfg.load(GOLDEN / "graphs" / f"doitgen.{variant}.json")
    ex = GpuExecutor(g, syms)
    try:
        assert any(sp.mode == "contract" for sp in ex.specs.values())
    finally:
        ex.close()
    rng = np.random.default_rng(6)
    A = rng.uniform(-1, 1, (8, 12, NP))
    C4 = rng.uniform(-1, 1, (NP, NP))
    out = interpret(g, ExecContext(bindings=dict(syms)).bind_inputs(
        {"A": A, "C4": C4, "out": np.full((8, 12, NP), np.nan)}))
    ref = np.einsum("rqs,sp->rqp", A, C4)
    assert rel_err(out["out"], ref) <= 1e-12
