"""dev tool: libb2 NCCL plumbing on one GPU (init, self p2p eager, self p2p captured)."""
import ctypes, faulthandler, os, sys, time
sys.path.insert(0, '.')
faulthandler.dump_traceback_later(40, exit=True)
import numpy as np
import torch.distributed as tdist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29551")
tdist.init_process_group("gloo", rank=0, world_size=1)
from paper_2107_00555_b200 import dist, runtime as rt
rt.device(0); L = rt.lib()
t = time.time(); comm = dist.NcclComm(0, 1); print("init", time.time() - t, flush=True)
n = 1 << 16
a = np.arange(n, dtype=np.float64)
pa, pb, s = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
rt.check(L.b2_malloc(ctypes.byref(pa), n * 8)); rt.check(L.b2_malloc(ctypes.byref(pb), n * 8))
rt.check(L.b2_stream_create(ctypes.byref(s)))
rt.check(L.b2_memcpy_h2d(pa, a.ctypes.data, n * 8, s)); rt.check(L.b2_stream_sync(s))
mode = sys.argv[1] if len(sys.argv) > 1 else "eager"
if mode == "capture":
    rt.check(L.b2_capture_begin(s))
comm.p2p([(True, 0, pa.value, n * 8), (False, 0, pb.value, n * 8)], s.value)
print("p2p issued", flush=True)
if mode == "capture":
    ge = ctypes.c_void_p(); rt.check(L.b2_capture_end(s, ctypes.byref(ge))); print("captured", flush=True)
    rt.check(L.b2_graph_launch(ge, s))
out = np.empty(n); rt.check(L.b2_memcpy_d2h(out.ctypes.data, pb, n * 8, s)); rt.check(L.b2_stream_sync(s))
print(mode, "ok" if np.array_equal(out, a) else "MISMATCH", flush=True)
