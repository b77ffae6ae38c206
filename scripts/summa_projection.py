"""Per-rank compute work of SUMMA 16384^3 on the squarest grids (2x1, 2x2,
4x2), measured on ONE GPU (no rank waits on another): rank (i, j) owns
A (M/Pr x K/Pc), B (K/Pr x N/Pc), C (M/Pr x N/Pc) and multiplies L =
lcm(Pr, Pc) panel products (M/Pr x K/L) @ (K/L x N/Pc) into C.
f64: libb2 DMMA DGEMM per panel.  f32: the local blocks are split into
3xTF32 hi/lo operands ONCE per call (b2_tf32_split_a / _bt, panel-major so a
panel is one contiguous broadcast buffer), then one b2_gemm_f32_presplit per
panel.  T1 = the same call on one GPU (b2_gemm_f64 / b2_gemm_f32 16384^3).
Compute-side efficiency = T1 / (P * T_rank), both timed sustained (1.5 s of
back-to-back calls each, T1 re-timed next to every grid: the GEMMs run
power-capped); the panel broadcasts overlap the
previous panel's GEMM in the multi-GPU runner and are not part of this
projection."""
import ctypes
import json
import math
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_2107_00555_b200 import runtime as rt  # noqa: E402

rt.device(0)
L = rt.lib()
n = 16384
out = {}
WHICH = sys.argv[1].split(",") if len(sys.argv) > 1 else ["f64", "f32"]


def alloc(nbytes, fill=None, dtype=None, shape=None, rng=None):
    p = ctypes.c_void_p()
    rt.check(L.b2_malloc(ctypes.byref(p), nbytes))
    if fill == "rand":
        h = rng.uniform(-1, 1, shape).astype(dtype)
        rt.check(L.b2_memcpy_h2d(p, h.ctypes.data, h.nbytes, None))
    else:
        rt.check(L.b2_memset(p, 0, nbytes, None))
    return p.value


s = ctypes.c_void_p()
rt.check(L.b2_stream_create(ctypes.byref(s)))
e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
L.b2_event_create(ctypes.byref(e0))
L.b2_event_create(ctypes.byref(e1))


def timed(fn, secs=1.5):
    """Sustained time of one call: fn repeated for `secs` seconds (the part
    settles at its power-capped clocks), median of the second half of the
    per-call CUDA-event times."""
    import time

    ts = []
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < secs or len(ts) < 4:
        L.b2_event_record(e0, s)
        fn()
        L.b2_event_record(e1, s)
        ms = ctypes.c_float()
        rt.check(L.b2_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
        ts.append(ms.value)
    return float(np.median(ts[len(ts) // 2:]))


rng = np.random.default_rng(0)
for dtype in WHICH:
    esz = 8 if dtype == "f64" else 4
    npd = np.float64 if dtype == "f64" else np.float32
    A = alloc(n * n * esz, "rand", npd, (n, n), rng)
    B = alloc(n * n * esz, "rand", npd, (n, n), rng)
    C = alloc(n * n * esz)
    if dtype == "f64":
        def full():
            rt.check(L.b2_gemm_f64(n, n, n, A, n, 1, B, n, 1, C, n, 1, 1, s))
    else:
        def full():
            rt.check(L.b2_gemm_f32(n, n, n, A, n, 1, B, n, 1, C, n, 1, 1, s))

    res = {}
    for (pr, pc) in ((2, 1), (2, 2), (4, 2)):
        P = pr * pc
        Lp = math.lcm(pr, pc)
        am, ak, bk, bn, kb = n // pr, n // pc, n // pr, n // pc, n // Lp
        if dtype == "f64":
            def rank():
                for _ in range(Lp):
                    rt.check(L.b2_gemm_f64(am, bn, kb, A, ak, 1, B, bn, 1, C, bn, 1, 1, s))
        else:
            kp = L.b2_tf32_split_cols(kb)
            pa = [alloc(am * kp * 4) for _ in range(Lp // pc)]
            pb = [alloc(bn * kp * 4) for _ in range(Lp // pr)]

            def rank():
                # split this rank's blocks once, panel by panel (contiguous
                # broadcast buffers), then one GEMM per received panel
                for la, p in enumerate(pa):
                    rt.check(L.b2_tf32_split_a(A + 4 * la * kb, ak, am, kb, p, s))
                for lb, p in enumerate(pb):
                    rt.check(L.b2_tf32_split_bt(B + 4 * lb * kb * bn, bn, kb, bn, p, s))
                for l in range(Lp):
                    rt.check(L.b2_gemm_f32_presplit(am, bn, kb, pa[l % len(pa)],
                                                    pb[l % len(pb)], C, bn, 1, s))
        # T1 re-timed right before each grid: both sides see the same
        # (power-capped) clocks
        t1 = timed(full)
        t = timed(rank)
        res[f"{pr}x{pc}"] = {"rank_ms": t, "T1_ms": t1, "efficiency": t1 / (P * t)}
        print(json.dumps({"dtype": dtype, "grid": f"{pr}x{pc}", "rank_ms": t, "T1_ms": t1,
                          "projected_efficiency": t1 / (P * t)}), flush=True)
        if dtype == "f32":
            for p in pa + pb:
                L.b2_free(p)
    out[dtype] = res
    for p in (A, B, C):
        L.b2_free(p)
json.dump(out, open("gpurun_out/summa_projection.json", "w"), indent=1)
