"""Kernel-level GPU checks at sizes beyond the golden fixtures: the DMMA
DGEMM (MATMUL 2D@2D), the rowpass BLAS-2 family and the stencil sweeps at
BASELINE config sizes against the CPU oracle ports (numpy / C)."""

import numpy as np
import pytest

from conftest import GOLDEN, rel_err

pytestmark = pytest.mark.gpu


def _run(name, syms, inputs):
    from paper_2107_00555_b200 import ExecContext, interpret, sdfg

    g = sdfg.load(GOLDEN / "graphs" / f"{name}.json")
    return interpret(g, ExecContext(bindings=dict(syms)).bind_inputs(inputs))


@pytest.mark.parametrize("M,K,N", [(300, 256, 512), (257, 129, 383), (1024, 2048, 768)])
def test_dgemm_dmma_vs_numpy(M, K, N):
    rng = np.random.default_rng(M + K + N)
    A = rng.uniform(-1, 1, (M, K))
    B = rng.uniform(-1, 1, (K, N))
    out = _run("matmul.raw", {"M": M, "K": K, "N": N}, {"A": A, "B": B, "C": np.zeros((M, N))})
    assert rel_err(out["C"], A @ B) <= 1e-12


@pytest.mark.parametrize("name,syms", [("atax.raw", {"M": 3000, "N": 2500}),
                                       ("bicg.raw", {"N": 2700, "M": 3100}),
                                       ("gemver.raw", {"N": 2048})])
def test_blas2_rowpass_vs_numpy_port(name, syms):
    from oracle import kernels_np as K

    rng = np.random.default_rng(5)
    from paper_2107_00555_b200 import sdfg, symexpr

    g = sdfg.load(GOLDEN / "graphs" / f"{name}.json")
    inputs = {}
    for n, c in g.containers.items():
        if not c.transient:
            shape = tuple(symexpr.evaluate(d, syms) for d in c.shape)
            inputs[n] = rng.uniform(-1, 1, shape) if shape else float(rng.uniform(0.5, 1.5))
    out = _run(name, syms, {k: np.array(v, copy=True) for k, v in inputs.items()})
    fn = getattr(K, name.split(".")[0])
    import inspect
    ref = fn(*[np.array(inputs[p], copy=True) if np.ndim(inputs[p]) else inputs[p]
               for p in inspect.signature(fn).parameters])
    for k, v in ref.items():
        assert rel_err(out[k], v) <= 1e-12, k


def test_heat3d_config_size_bitwise_vs_c_oracle():
    """heat_3d at the full N=400 (few steps): bitwise equal to the C oracle."""
    from oracle import kernels_np as K

    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (400, 400, 400))
    B = rng.uniform(-1, 1, (400, 400, 400))
    out = _run("heat_3d.raw", {"N": 400, "TSTEPS": 4}, {"A": A.copy(), "B": B.copy()})
    K.heat_3d_c(A, B, 4)
    assert np.array_equal(out["A"], A) and np.array_equal(out["B"], B)


def test_jacobi2d_config_size_bitwise_vs_c_oracle():
    from oracle import kernels_np as K

    rng = np.random.default_rng(1)
    A = rng.uniform(-1, 1, (2000, 2000))
    B = rng.uniform(-1, 1, (2000, 2000))
    out = _run("jacobi_2d.raw", {"N": 2000, "TSTEPS": 100}, {"A": A.copy(), "B": B.copy()})
    K.jacobi_2d_c(A, B, 100)
    assert np.array_equal(out["A"], A) and np.array_equal(out["B"], B)


@pytest.mark.parametrize("M,K,N", [(512, 256, 384), (300, 200, 452), (1024, 1000, 768)])
def test_sgemm_vs_numpy(M, K, N):
    """f32 GEMM (SUMMA f32 config): rtol 1e-5 (norm-wise) against an f64
    product of the f32-rounded inputs, and no less accurate
    than numpy's own f32 matmul (element-wise errors of an f32 K-term sum
    grow with K, so an element-wise 1e-5 bound does not hold for either)."""
    import ctypes

    from paper_2107_00555_b200 import runtime as rt

    rt.device(0)
    L = rt.lib()
    rng = np.random.default_rng(M + N)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ptr = []
    for arr in (A, B, np.zeros((M, N), np.float32)):
        p = ctypes.c_void_p()
        rt.check(L.b2_malloc(ctypes.byref(p), arr.nbytes))
        rt.check(L.b2_memcpy_h2d(p, arr.ctypes.data, arr.nbytes, None))
        ptr.append(p)
    rt.check(L.b2_gemm_f32(M, N, K, ptr[0], K, 1, ptr[1], N, 1, ptr[2], N, 1, 0, None))
    C = np.empty((M, N), np.float32)
    rt.check(L.b2_memcpy_d2h(C.ctypes.data, ptr[2], C.nbytes, None))
    rt.check(L.b2_device_sync())
    ref = A.astype(np.float64) @ B.astype(np.float64)
    ours = np.linalg.norm(C - ref) / np.linalg.norm(ref)
    assert ours <= 1e-5
    npf32 = np.linalg.norm((A @ B).astype(np.float64) - ref) / np.linalg.norm(ref)
    assert ours <= 10 * npf32 + 1e-7
    for p in ptr:
        L.b2_free(p)


@pytest.mark.parametrize("M,K,N,acc", [(1024, 512, 1024, False), (1000, 300, 777, True),
                                       (256, 4096, 512, False)])
def test_tc_sgemm_3xtf32_vs_numpy(M, K, N, acc):
    """tcgen05 3xTF32 path of b2_gemm_f32 (large problems), incl. ragged tiles
    (TMA zero fill, guarded epilogue) and WCR add: same bar as above."""
    import ctypes

    from paper_2107_00555_b200 import runtime as rt

    rt.device(0)
    L = rt.lib()
    rng = np.random.default_rng(M * 7 + N)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32) if acc else np.zeros((M, N), np.float32)
    ptr = []
    for arr in (A, B, C0):
        p = ctypes.c_void_p()
        rt.check(L.b2_malloc(ctypes.byref(p), arr.nbytes))
        rt.check(L.b2_memcpy_h2d(p, arr.ctypes.data, arr.nbytes, None))
        ptr.append(p)
    n0 = L.b2_launch_count()
    rt.check(L.b2_gemm_f32(M, N, K, ptr[0], K, 1, ptr[1], N, 1, ptr[2], N, 1,
                           1 if acc else 0, None))
    assert L.b2_launch_count() - n0 >= 3  # split A, split B, tensor-core GEMM
    C = np.empty((M, N), np.float32)
    rt.check(L.b2_memcpy_d2h(C.ctypes.data, ptr[2], C.nbytes, None))
    rt.check(L.b2_device_sync())
    ref = C0.astype(np.float64) + A.astype(np.float64) @ B.astype(np.float64)
    ours = np.linalg.norm(C - ref) / np.linalg.norm(ref)
    assert ours <= 1e-5, ours
    npf32 = np.linalg.norm((C0 + A @ B).astype(np.float64) - ref) / np.linalg.norm(ref)
    assert ours <= 10 * npf32 + 1e-7
    for p in ptr:
        L.b2_free(p)


@pytest.mark.parametrize("N,H,SM", [(2, 3, 1), (2, 3, 33), (1, 2, 64), (3, 1, 100)])
def test_softmax_fold_and_rowred_vs_numpy_port(N, H, SM):
    """softmax raw graph: the max loop runs as a warp fold (incl. zero-trip and
    ragged-lane cases), the exp/sum map in row-reduction mode with the divide
    fused as its epilogue (ragged rows of 33 / 100: partial register rows)."""
    from oracle import kernels_np as K

    rng = np.random.default_rng(SM)
    x = rng.uniform(-1, 1, (N, H, SM, SM))
    out = _run("softmax.raw", {"N": N, "H": H, "SM": SM}, {"x": x, "out": np.zeros_like(x)})
    ref = np.empty_like(x)
    K.softmax(x.copy(), ref)
    assert rel_err(out["out"], ref) <= 1e-12


def test_softmax_divide_runs_as_row_epilogue():
    """The row-reduction epilogue fusion is what runs: the divide map is not
    launched on its own and ex never gets a kernel store."""
    from paper_2107_00555_b200 import sdfg
    from paper_2107_00555_b200.machine import GpuExecutor

    g = sdfg.load(GOLDEN / "graphs" / "softmax.raw.json")
    ex = GpuExecutor(g, {"N": 2, "H": 3, "SM": 64})
    try:
        assert len(ex.epi_skip) == 1
        fused = [sp for sp in ex.specs.values() if getattr(sp, "epilogue", None) is not None]
        assert len(fused) == 1 and "c_ex[" not in fused[0].source
    finally:
        ex.close()


def test_run_twice_bitwise_deterministic():
    """run_twice_determinism (interp.py:153) on chunked reductions: the
    go_fast trace (12000-term sum into one scalar) is folded in chunk order
    by a second kernel, so repeated runs are bitwise identical."""
    from paper_2107_00555_b200 import ExecContext, interpret, run_twice_determinism, sdfg

    g = sdfg.load(GOLDEN / "graphs" / "go_fast.pipe.json")
    rng = np.random.default_rng(9)
    a = rng.uniform(-1, 1, (3000, 3000))
    ctx = ExecContext(bindings={"N": 3000}).bind_inputs({"a": a, "out": np.zeros_like(a)})
    assert run_twice_determinism(g, ctx)
    outs = [interpret(g, ExecContext(bindings={"N": 3000}).bind_inputs(
        {"a": a, "out": np.zeros_like(a)}))["out"] for _ in range(3)]
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("name,syms,shape", [("heat_3d.raw", {"N": 24, "TSTEPS": 4}, (24, 24, 24)),
                                             ("jacobi_2d.raw", {"N": 40, "TSTEPS": 5}, (40, 40))])
def test_dead_interior_inputs_upload_only_faces(name, syms, shape):
    """B's interior is overwritten before it is read, so only its boundary
    faces are uploaded: NaNs in the input interior never reach the result."""
    from oracle import kernels_np as K
    from paper_2107_00555_b200 import sdfg
    from paper_2107_00555_b200.machine import GpuExecutor

    g = sdfg.load(GOLDEN / "graphs" / f"{name}.json")
    ex = GpuExecutor(g, syms)
    assert ex.shell_only == {"B"}
    rng = np.random.default_rng(1)
    A = rng.uniform(-1, 1, shape)
    B = rng.uniform(-1, 1, shape)
    Bn = B.copy()
    Bn[(slice(1, -1),) * len(shape)] = np.nan
    out = _run(name, syms, {"A": A.copy(), "B": Bn})
    (K.heat_3d_c if len(shape) == 3 else K.jacobi_2d_c)(A, B, syms["TSTEPS"])
    assert np.array_equal(out["A"], A) and np.array_equal(out["B"], B)
    ex.close()


def test_conv2d_register_blocked_reduction_bitwise(monkeypatch):
    """conv2d_bias's 7-D WCR map with the output channel register-blocked
    (each thread owns all CO accumulators, codegen._reduce_loop_blocked):
    bitwise equal to the thread-per-output schedule, and to the oracle."""
    from oracle import kernels_np as K
    from paper_2107_00555_b200 import codegen

    syms = {"NB": 2, "H": 160, "W": 160, "CI": 3, "CO": 16, "K": 20, "HO": 141, "WO": 141}
    rng = np.random.default_rng(21)
    x = {"inp": rng.uniform(-1, 1, (2, 160, 160, 3)), "w": rng.uniform(-1, 1, (20, 20, 3, 16)),
         "bias": rng.uniform(-1, 1, 16), "out": np.zeros((2, 141, 141, 16))}
    outs = {}
    for rb in (16, 0):
        monkeypatch.setattr(codegen, "RED_BLOCK", rb)
        outs[rb] = _run("conv2d_bias.raw", syms, {k: v.copy() for k, v in x.items()})["out"]
    assert np.array_equal(outs[16], outs[0])
    ref = np.zeros_like(x["out"])
    K.conv2d_bias(x["inp"], x["w"], x["bias"], ref)
    assert rel_err(outs[16], ref) <= 1e-12


def test_init_fill_fused_into_reduction_bitwise(monkeypatch):
    """nbody's get_acc: ``acc[:] = 0.0`` followed by the pair-force WCR map.
    With the fill folded into the reduction's initial value (one kernel
    fewer per call) the run is bitwise equal to launching both, with the
    same counters."""
    from paper_2107_00555_b200 import ExecContext, interpret, machine, sdfg

    g = sdfg.load(GOLDEN / "graphs" / "nbody.raw.json")
    rng = np.random.default_rng(4)
    n = 64
    x = {"mass": rng.uniform(0.5, 1.5, n), "pos": rng.uniform(-1, 1, (n, 3)),
         "vel": rng.uniform(-1, 1, (n, 3)), "acc": np.zeros((n, 3)), "E": np.zeros(2),
         "G": 1.0, "softening": 0.1, "dt": 0.01}
    res = {}
    for mode in (True, False):
        monkeypatch.setattr(machine, "INIT_FUSION", mode)
        ctx = ExecContext(bindings={"N": n, "NT": 7}).bind_inputs(
            {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in x.items()})
        out = interpret(g, ctx)
        res[mode] = (out, ctx.counters.as_dict())
    for k in ("pos", "vel", "acc", "E"):
        assert np.array_equal(res[True][0][k], res[False][0][k]), k
    assert res[True][1] == res[False][1]


def test_fully_overwritten_transients_not_zeroed():
    """atax's tmp0 = A @ x is written in full by the row pass before anything
    reads it, so the per-call zeroing (interp.py:220-221) is skipped; the
    result still matches the port."""
    from oracle import kernels_np as K
    from paper_2107_00555_b200 import sdfg
    from paper_2107_00555_b200.machine import GpuExecutor

    g = sdfg.load(GOLDEN / "graphs" / "atax.raw.json")
    ex = GpuExecutor(g, {"M": 300, "N": 200})
    assert ex.zero_skip == {"tmp0"}
    ex.close()
    rng = np.random.default_rng(2)
    A, x = rng.uniform(-1, 1, (300, 200)), rng.uniform(-1, 1, 200)
    out = _run("atax.raw", {"M": 300, "N": 200}, {"A": A, "x": x, "y": np.zeros(200)})
    ref = K.atax(A.copy(), x.copy(), np.zeros(200))
    assert rel_err(out["y"], ref["y"]) <= 1e-12


def test_tf32_presplit_gemm_equals_gemm_f32():
    """b2_tf32_split_a / _bt + b2_gemm_f32_presplit (SUMMA f32's split-once
    path) is the same computation as b2_gemm_f32: bitwise equal output."""
    import ctypes

    from paper_2107_00555_b200 import runtime as rt

    L = rt.lib()
    M, N, K = 512, 768, 640
    rng = np.random.default_rng(9)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    kp = L.b2_tf32_split_cols(K)
    sizes = (A.nbytes, B.nbytes, M * N * 4, M * N * 4, M * kp * 4, N * kp * 4)
    ptr = [ctypes.c_void_p() for _ in sizes]
    for p, nb in zip(ptr, sizes):
        rt.check(L.b2_malloc(ctypes.byref(p), nb))
    try:
        rt.check(L.b2_memcpy_h2d(ptr[0], A.ctypes.data, A.nbytes, None))
        rt.check(L.b2_memcpy_h2d(ptr[1], B.ctypes.data, B.nbytes, None))
        rt.check(L.b2_gemm_f32(M, N, K, ptr[0], K, 1, ptr[1], N, 1, ptr[2], N, 1, 0, None))
        rt.check(L.b2_tf32_split_a(ptr[0], K, M, K, ptr[4], None))
        rt.check(L.b2_tf32_split_bt(ptr[1], N, K, N, ptr[5], None))
        rt.check(L.b2_gemm_f32_presplit(M, N, K, ptr[4], ptr[5], ptr[3], N, 0, None))
        c1 = np.empty((M, N), np.float32)
        c2 = np.empty((M, N), np.float32)
        rt.check(L.b2_memcpy_d2h(c1.ctypes.data, ptr[2], c1.nbytes, None))
        rt.check(L.b2_memcpy_d2h(c2.ctypes.data, ptr[3], c2.nbytes, None))
        rt.check(L.b2_device_sync())
        assert np.array_equal(c1, c2)
        ref = A.astype(np.float64) @ B.astype(np.float64)
        assert np.linalg.norm(c2 - ref) / np.linalg.norm(ref) <= 1e-5
    finally:
        for p in ptr:
            L.b2_free(p)
