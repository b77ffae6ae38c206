"""Dev probe: time b2_gemm_f32 (tcgen05 3xTF32 path) at n^3 with CUDA events."""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2107_00555_b200 import runtime as rt

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
M, N, K = (int(x) for x in sys.argv[3].split("x")) if len(sys.argv) > 3 else (n, n, n)
rt.device(0)
L = rt.lib()
rng = np.random.default_rng(0)
ptr = []
for shape in ((M, K), (K, N), (M, N)):
    a = rng.uniform(-1, 1, shape).astype(np.float32)
    p = ctypes.c_void_p()
    rt.check(L.b2_malloc(ctypes.byref(p), a.nbytes))
    rt.check(L.b2_memcpy_h2d(p, a.ctypes.data, a.nbytes, None))
    ptr.append(p)
s = ctypes.c_void_p()
rt.check(L.b2_stream_create(ctypes.byref(s)))
e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
L.b2_event_create(ctypes.byref(e0)); L.b2_event_create(ctypes.byref(e1))
for r in range(reps):
    L.b2_event_record(e0, s)
    rt.check(L.b2_gemm_f32(M, N, K, ptr[0], K, 1, ptr[1], N, 1, ptr[2], N, 1, 1, s))
    L.b2_event_record(e1, s)
    ms = ctypes.c_float()
    rt.check(L.b2_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
    print(f"rep {r}: {ms.value:.3f} ms  {2 * M * N * K / ms.value / 1e9:.1f} TFLOP/s", flush=True)
