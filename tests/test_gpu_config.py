"""Config-size parity: every BASELINE.json configuration, at its full size,
through the public ``interpret()`` on the B200, against digests of the
REFERENCE's own outputs (tests/golden/make_config_digests.py ran
``sdfgkit.frontend.evaluate_program`` on the same seeded inputs; three
NPBench programs use the bitwise-pinned numpy port, see the generator).

Criteria, per output (tolerances written here, north_star: rtol 1e-12 f64,
1e-5 f32):
* BITWISE outputs (fixed op order on both sides: stencils, the elementwise
  gemver update): sha256 of the whole array equal to the reference's.
* fixed-order outputs: rel_err (pkg/tests/conftest.py:85-93, floor 1) at
  the digest points <= rtol and row sums within rtol (relative to the row's
  sum of magnitudes).
* re-associated sums (BLAS-2 products, MatMul), where the reference's own
  BLAS result is itself ~eps * sum|terms| away from the truth: rel_err
  against ``exact`` (an 80-bit evaluation of the same chain) <= rtol or no
  larger than the reference's own rel_err against it, AND
  the exact-sum criterion |gpu - exact| <= |oracle - exact| + 4 eps terms
  per element (``terms`` = the chain's first-order rounding magnitude,
  sum |terms|); rel_err against the oracle is reported beside.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

import config_digest as CD
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CFG = GOLDEN / "config"
CONFIGS = sorted(p.stem for p in CFG.glob("*.json")) if CFG.is_dir() else []

# (conv2d_bias runs on the FP64 tensor path since round 2: DMMA fuses the
# multiply-adds, so its result is within rtol, no longer bitwise)
BITWISE = {"jacobi_2d": {"A", "B"}, "heat_3d": {"A", "B"}, "gemver": {"A"}}
F64_RTOL = 1e-12
F32_RTOL = 1e-5


def _entry(name):
    return json.loads((CFG / f"{name}.json").read_text())


def _inputs(e, blob=None):
    if e.get("inputs") == "stored":
        return {k[3:]: (blob[k] if blob[k].ndim else float(blob[k]))
                for k in blob.files if k.startswith("in/")}
    shapes = {k: tuple(v) for k, v in e["shapes"].items()}
    return CD.make_inputs(e["params"], shapes, e["seed"], round_f32=tuple(e["round_f32"]))


def _run(name, e, inputs):
    if name == "matmul_f32":
        return {"C": _gemm_f32(inputs["A"], inputs["B"], precise=True)}
    from paper_2107_00555_b200 import ExecContext, interpret, sdfg

    g = sdfg.load(GOLDEN / "graphs" / f"{e['graph']}.json")
    ctx = ExecContext(bindings=dict(e["symbols"])).bind_inputs(inputs)
    out = interpret(g, ctx)
    _free_cache()
    return out


def _free_cache():
    """Config-size executors hold GBs of HBM: drop them between configs."""
    from paper_2107_00555_b200 import machine

    while machine._exec_cache:
        machine._exec_cache.popitem()[1].close()


def _gemm_f32(A, B, precise: bool):
    """The f32 MatMul config through the C ABI; the reference has no f32 type
    (SURVEY.md §8c), so the expectation is the f64 product of the f32-rounded
    inputs.  precise: b2_gemm_f32_f64acc (f64 products / accumulation, one
    rounding); else b2_gemm_f32 (tcgen05 3xTF32, fp32 accumulation)."""
    import ctypes

    from paper_2107_00555_b200 import runtime as rt

    L = rt.lib()
    M, K = A.shape
    N = B.shape[1]
    a = np.ascontiguousarray(A, dtype=np.float32)
    b = np.ascontiguousarray(B, dtype=np.float32)
    c = np.empty((M, N), dtype=np.float32)
    ptr = [ctypes.c_void_p() for _ in range(3)]
    for p, n in zip(ptr, (a.nbytes, b.nbytes, c.nbytes)):
        rt.check(L.b2_malloc(ctypes.byref(p), n))
    try:
        rt.check(L.b2_memcpy_h2d(ptr[0], a.ctypes.data, a.nbytes, None))
        rt.check(L.b2_memcpy_h2d(ptr[1], b.ctypes.data, b.nbytes, None))
        if precise:
            rt.check(L.b2_gemm_f32_f64acc(M, N, K, ptr[0], K, ptr[1], N, ptr[2], N, 0, None))
        else:
            rt.check(L.b2_gemm_f32(M, N, K, ptr[0], K, 1, ptr[1], N, 1, ptr[2], N, 1, 0, None))
        rt.check(L.b2_memcpy_d2h(c.ctypes.data, ptr[2], c.nbytes, None))
        rt.check(L.b2_stream_sync(None))
    finally:
        for p in ptr:
            L.b2_free(p)
    return c.astype(np.float64)


CHAOTIC = {"nbody"}  # 1000 leapfrog steps: a 1-ulp input change moves every output O(1)


@pytest.mark.parametrize("name", [c for c in CONFIGS if c not in CHAOTIC])
def test_config_parity(name):
    e = _entry(name)
    blob = np.load(CFG / f"{name}.npz")
    inputs = _inputs(e, blob)
    out = _run(name, e, inputs)
    rtol = F32_RTOL if name == "matmul_f32" else F64_RTOL
    report, fails = {}, []
    for k in e["outputs"]:
        ref = CD.unpack(blob, k)
        got = np.asarray(out[k], dtype=np.float64)
        assert tuple(got.shape) == tuple(ref["shape"]), (k, got.shape)
        same = CD.sha(got) == bytes(ref["sha256"])
        if k in BITWISE.get(name, ()) and not same:
            fails.append(f"{k}: not bitwise equal to the reference")
        vals = got.reshape(-1)[CD.picks(got.size)]
        err = CD.rel_err(vals, ref["values"])
        rep = {"bitwise": same, "rel_err_vs_oracle": err}
        has_exact = f"{k}/exact" in blob.files
        if has_exact:
            # re-associated sums: the oracle itself carries ~eps sum|terms|
            # of rounding (OpenBLAS), so rtol is held against the exact
            # value; the oracle's own distance to it is reported beside
            exact = blob[f"{k}/exact"].astype(np.longdouble) + blob[f"{k}/exact_lo"]
            ex64 = exact.astype(np.float64)
            err_x = CD.rel_err(vals, ex64)
            err_o = CD.rel_err(ref["values"], ex64)
            rep.update(rel_err_vs_exact=err_x, oracle_rel_err_vs_exact=err_o)
            if not (err_x <= rtol or err_x <= err_o):
                fails.append(f"{k}: rel_err vs exact {err_x:.3e} > {rtol} and > the "
                             f"reference's own {err_o:.3e}")
        elif not err <= rtol:
            fails.append(f"{k}: rel_err {err:.3e} > {rtol}")
        if "rowsum" in ref and not has_exact:
            rs = got.reshape(got.shape[0], -1).sum(axis=1)
            scale = np.maximum(np.abs(got).reshape(got.shape[0], -1).sum(axis=1), 1.0)
            with np.errstate(invalid="ignore"):
                d = np.abs(rs - ref["rowsum"]) / scale
            d = np.where(np.isnan(rs) & np.isnan(ref["rowsum"]), 0.0, d)  # 0/0 bins
            rerr = float(np.max(np.nan_to_num(d, nan=np.inf)))
            rep["rowsum_rel"] = rerr
            if not rerr <= rtol:
                fails.append(f"{k}: row-sum rel {rerr:.3e} > {rtol}")
        if has_exact and name != "matmul_f32":
            ok, ratio, eg, eo = CD.exact_criterion(vals, ref["values"], exact,
                                                   blob[f"{k}/terms"])
            rep.update(exact_ratio=ratio, gpu_vs_exact=eg, oracle_vs_exact=eo)
            if not ok:
                fails.append(f"{k}: exact-sum criterion ratio {ratio:.3f} > 1")
        report[k] = rep
    print(name, json.dumps(report))
    assert not fails, (name, fails, report)


def test_matmul_f32_tensor_core_vs_host_sgemm():
    """The throughput f32 path (tcgen05 3xTF32, fp32 accumulation, the SUMMA
    f32 kernel) at the config size 16384^3.  No fp32-accumulating GEMM meets
    an element-wise rtol 1e-5 (floor 1) at K = 16384 — the host's own sgemm
    misses it by ~6x on the same data — so this path is held to: norm-wise
    error <= 1e-5, and over a 256-row band of C its max and RMS element
    errors against the f64 product within 2x the host sgemm's (measured:
    1.2x / 1.4x).  The accurate f32 path (test_config_parity[matmul_f32])
    meets rtol 1e-5 element-wise."""
    e = _entry("matmul_f32")
    inputs = _inputs(e)
    A, B = inputs["A"], inputs["B"]
    C = _gemm_f32(A, B, precise=False)
    band = slice(0, 256)
    exact = A[band] @ B
    host = (A[band].astype(np.float32) @ B.astype(np.float32)).astype(np.float64)
    eg = np.abs(C[band] - exact) / np.maximum(np.abs(exact), 1.0)
    eh = np.abs(host - exact) / np.maximum(np.abs(exact), 1.0)
    blob = np.load(CFG / "matmul_f32.npz")
    ref = CD.unpack(blob, "C")
    vals = C.reshape(-1)[CD.picks(C.size)]
    normwise = float(np.linalg.norm(vals - ref["values"]) / np.linalg.norm(ref["values"]))
    rep = {"normwise": normwise, "gpu_max": float(eg.max()), "host_max": float(eh.max()),
           "gpu_rms": float(np.sqrt((eg ** 2).mean())), "host_rms": float(np.sqrt((eh ** 2).mean()))}
    print("matmul_f32 tensor-core", json.dumps(rep))
    assert normwise <= F32_RTOL, rep
    assert rep["gpu_max"] <= 2 * rep["host_max"] and rep["gpu_rms"] <= 2 * rep["host_rms"], rep


@pytest.mark.skipif("nbody" not in CONFIGS, reason="no nbody digest")
def test_nbody_preset_energy():
    """nbody at the NPBench preset (N=100, 1000 steps, NPBench init).  The
    trajectory is chaotic — perturbing one input coordinate by 1 ulp changes
    the reference's own outputs by O(1) after 1000 steps — so element-wise
    parity is checked on the 10-step config (nbody_short, rtol 1e-12) and
    here the run is held to what a faithful integrator must preserve: the
    total energy E[0] + E[1] agrees with the reference's to within 10x the
    reference's own drift from the initial energy, and every output is
    finite."""
    e = _entry("nbody")
    blob = np.load(CFG / "nbody.npz")
    inputs = _inputs(e, blob)
    out = _run("nbody", e, inputs)
    ref = CD.unpack(blob, "E")["values"]
    e0 = _run("nbody_e0", dict(e, symbols=dict(e["symbols"], NT=0)), dict(inputs))["E"]
    drift = abs((ref[0] + ref[1]) - (e0[0] + e0[1]))
    got = float(out["E"][0] + out["E"][1])
    rep = {"E_ref": float(ref[0] + ref[1]), "E_gpu": got, "E_initial": float(e0[0] + e0[1]),
           "ref_drift": float(drift)}
    print("nbody", json.dumps(rep))
    assert all(np.all(np.isfinite(v)) for v in out.values())
    assert abs(got - (ref[0] + ref[1])) <= 10 * drift + 1e-12, rep
