"""TF32x3 presplit GEMM rate at the SUMMA panel shapes (CUDA events, best
and median of 5), to compare kernel revisions."""
import ctypes
import json
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_2107_00555_b200 import runtime as rt  # noqa: E402

rt.device(0)
L = rt.lib()
s = ctypes.c_void_p()
rt.check(L.b2_stream_create(ctypes.byref(s)))
e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
L.b2_event_create(ctypes.byref(e0))
L.b2_event_create(ctypes.byref(e1))


def alloc(n):
    p = ctypes.c_void_p()
    rt.check(L.b2_malloc(ctypes.byref(p), n))
    rt.check(L.b2_memset(p, 0, n, None))
    return p.value


for (M, N, K) in ((16384, 16384, 16384), (8192, 16384, 8192), (8192, 8192, 8192),
                  (4096, 8192, 4096), (4096, 4096, 4096)):
    kp = L.b2_tf32_split_cols(K)
    A = alloc(M * kp * 4)
    B = alloc(N * kp * 4)
    C = alloc(M * N * 4)
    ts = []
    for r in range(6):
        L.b2_event_record(e0, s)
        rt.check(L.b2_gemm_f32_presplit(M, N, K, A, B, C, N, 1, s))
        L.b2_event_record(e1, s)
        ms = ctypes.c_float()
        rt.check(L.b2_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
        ts.append(ms.value)
    ts = ts[1:]
    fl = 2.0 * M * N * K
    print(json.dumps({"M": M, "N": N, "K": K, "best_ms": min(ts), "med_ms": float(np.median(ts)),
                      "TFLOPs_best": fl / min(ts) / 1e9, "TFLOPs_med": fl / float(np.median(ts)) / 1e9}))
    for p in (A, B, C):
        L.b2_free(p)
