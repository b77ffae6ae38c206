"""Quick device timing of one golden graph at a given size (dev tool)."""
import ctypes, json, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2107_00555_b200 import sdfg, runtime as rt
from paper_2107_00555_b200.machine import GpuExecutor

name = sys.argv[1]
syms = json.loads(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g = sdfg.load(f'tests/golden/graphs/{name}.json')
t0 = time.time()
ex = GpuExecutor(g, syms)
print(f"plan+compile {time.time()-t0:.2f}s  ops={len(ex.planner.all_ops)}", flush=True)
rng = np.random.default_rng(0)
inputs = {}
for n, c in g.containers.items():
    if not c.transient:
        shape = ex.buf.shape[n]
        inputs[n] = rng.uniform(-1, 1, size=shape) if shape else np.float64(rng.uniform(0.5, 1.5))
ex.prepare_inputs(inputs); ex.sync()
L = rt.lib()
e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
L.b2_event_create(ctypes.byref(e0)); L.b2_event_create(ctypes.byref(e1))
for r in range(reps):
    t = time.time()
    L.b2_event_record(e0, ex.stream)
    ex.run_device(first_call=(r == 0))
    L.b2_event_record(e1, ex.stream)
    ms = ctypes.c_float()
    rt.check(L.b2_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
    print(f"rep {r}: device {ms.value:.3f} ms  wall {1e3*(time.time()-t):.1f} ms  launches={ex.launches}", flush=True)
ex.check_flag()
prof = ex.profile_launches()
for k, (n, tot, npts) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print(f"  kernel {k}: {n} launches, {tot/n*1e3:.1f} us avg, {tot:.3f} ms total")
