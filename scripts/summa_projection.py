"""Per-rank GEMM work of SUMMA 16384^3 on the squarest grids (2x1, 2x2, 4x2)
measured on ONE GPU: each rank multiplies L = lcm(Pr, Pc) panel products of
(M/Pr x K/L) @ (K/L x N/Pc) into its C block (libb2 b2_gemm_f64 / f32, the
same calls dist.Summa makes); the panel broadcasts overlap the previous
panel's GEMM.  Compute-side efficiency = T1 / (P * T_rank)."""
import ctypes, json, math, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2107_00555_b200 import runtime as rt

rt.device(0)
L = rt.lib()
n = 16384
out = {}
WHICH = sys.argv[1].split(",") if len(sys.argv) > 1 else ["f64", "f32"]
for dtype, fn, esz in (("f64", L.b2_gemm_f64, 8), ("f32", L.b2_gemm_f32, 4)):
    if dtype not in WHICH:
        continue
    bufs = []
    rng = np.random.default_rng(0)
    for i, shape in enumerate(((n, n), (n, n), (n, n))):
        p = ctypes.c_void_p()
        rt.check(L.b2_malloc(ctypes.byref(p), shape[0] * shape[1] * esz))
        if i < 2:  # random operands: the tensor cores draw (and get clocked) like the bench
            h = rng.uniform(-1, 1, shape).astype(np.float64 if esz == 8 else np.float32)
            rt.check(L.b2_memcpy_h2d(p, h.ctypes.data, h.nbytes, None))
            del h
        else:
            rt.check(L.b2_memset(p, 0, shape[0] * shape[1] * esz, None))
        bufs.append(p)
    s = ctypes.c_void_p()
    rt.check(L.b2_stream_create(ctypes.byref(s)))
    e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
    L.b2_event_create(ctypes.byref(e0)); L.b2_event_create(ctypes.byref(e1))

    def run(M, N, K, panels):
        for rep in range(2):  # warm, then timed
            L.b2_event_record(e0, s)
            for l in range(panels):
                rt.check(fn(M, N, K, bufs[0], K, 1, bufs[1], N, 1, bufs[2], N, 1, 1, s))
            L.b2_event_record(e1, s)
            ms = ctypes.c_float()
            rt.check(L.b2_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
        return ms.value

    t1 = run(n, n, n, 1)
    res = {"1": t1}
    for (pr, pc) in ((2, 1), (2, 2), (4, 2)):
        P = pr * pc
        Lp = math.lcm(pr, pc)
        t = run(n // pr, n // pc, n // Lp, Lp)
        res[f"{pr}x{pc}"] = {"ms": t, "efficiency": t1 / (P * t)}
        print(json.dumps({"dtype": dtype, "grid": f"{pr}x{pc}", "rank_ms": t, "T1_ms": t1,
                          "projected_efficiency": t1 / (P * t)}), flush=True)
    out[dtype] = res
    for p in bufs:
        L.b2_free(p)
json.dump(out, open("gpurun_out/summa_projection.json", "w"), indent=1)
