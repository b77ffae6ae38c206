"""Dev probe: norm-wise error of b2_gemm_f32 (tcgen05 3xTF32) vs an f64
product, against numpy's f32 matmul, for growing K."""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2107_00555_b200 import runtime as rt

rt.device(0)
L = rt.lib()
for K in (1024, 4096, 16384):
    M, N = 512, 768
    rng = np.random.default_rng(K)
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
    e = np.linalg.norm(C - ref) / np.linalg.norm(ref)
    en = np.linalg.norm((A @ B).astype(np.float64) - ref) / np.linalg.norm(ref)
    em = np.max(np.abs(C - ref)) / np.max(np.abs(ref))
    print(f"K={K}: tc {e:.3e} (max {em:.3e})  numpy-f32 {en:.3e}", flush=True)
    for p in ptr:
        L.b2_free(p)
