"""b2_gemm_f64 rate (CUDA events, median of 3 after a warm call, random
operands) at 4096^3, 8192^3 and 16384^3 — for comparing DGEMM revisions."""
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
rng = np.random.default_rng(0)
for n in (4096, 8192, 16384):
    ptr = []
    for _ in range(2):
        h = rng.uniform(-1, 1, (n, n))
        p = ctypes.c_void_p()
        rt.check(L.b2_malloc(ctypes.byref(p), h.nbytes))
        rt.check(L.b2_memcpy_h2d(p, h.ctypes.data, h.nbytes, None))
        ptr.append(p.value)
    c = ctypes.c_void_p()
    rt.check(L.b2_malloc(ctypes.byref(c), n * n * 8))
    ts = []
    for r in range(4):
        L.b2_event_record(e0, s)
        rt.check(L.b2_gemm_f64(n, n, n, ptr[0], n, 1, ptr[1], n, 1, c, n, 1, 0, s))
        L.b2_event_record(e1, s)
        ms = ctypes.c_float()
        rt.check(L.b2_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
        ts.append(ms.value)
    med = float(np.median(ts[1:]))
    print(json.dumps({"n": n, "ms": med, "TFLOPs": 2.0 * n ** 3 / med / 1e9}), flush=True)
    for p in ptr + [c.value]:
        L.b2_free(p)
