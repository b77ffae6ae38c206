"""Per-rank work of the slab-decomposed heat_3d at P = 2/4/8 measured on ONE
GPU: rank r's local graph runs through the same executor, overlap split and
captured CUDA graph as under torchrun, with the NCCL transfer replaced by a
no-op (the exchange itself overlaps the interior sweep).  Reports the device
time per program run and the strong-scaling efficiency T1 / (P * T_rank)
this work implies.  (Evidence for the multi-GPU design on a 1-GPU pool; the
real multi-GPU number is the driver's SCALE run.)"""
import ctypes, json, sys
sys.path.insert(0, '.')
import numpy as np
import torch.distributed as tdist
import os, socket

from paper_2107_00555_b200 import dist, runtime as rt, sdfg
from bench import make_inputs

s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
tdist.init_process_group("gloo", rank=0, world_size=1)

N, T = 400, 100
syms = {"N": N, "TSTEPS": T}
g = sdfg.load("tests/golden/graphs/heat_3d.raw.json")
inputs = make_inputs(g, syms)


class _NoTransfer:
    def p2p(self, ops, stream):
        return sum(x[3] for x in ops if x[0])

    def close(self):
        pass


def time_runner(runner, reps=3):
    L = rt.lib()
    e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
    L.b2_event_create(ctypes.byref(e0)); L.b2_event_create(ctypes.byref(e1))
    runner.run(); runner.ex.sync()
    best = 1e30
    for _ in range(reps):
        L.b2_event_record(e0, runner.ex.stream)
        runner.run()
        L.b2_event_record(e1, runner.ex.stream)
        ms = ctypes.c_float()
        rt.check(L.b2_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
        best = min(best, ms.value)
    return best


res = {}
r1 = dist.SlabGpuRunner(g, syms, 0, 1, 0)
r1.load_inputs(inputs)
t1 = time_runner(r1)
res[1] = {"ms": t1}
print(json.dumps({"P": 1, "ms_per_run": t1}), flush=True)
for P in (2, 4, 8):
    worst = 0.0
    for rank in sorted({0, P // 2}):  # an edge rank and an interior rank
        r = dist.SlabGpuRunner.__new__(dist.SlabGpuRunner)
        # same construction as SlabGpuRunner.__init__ for (rank, P), transfer stubbed
        import torch
        from paper_2107_00555_b200.machine import GpuExecutor, InterpOptions
        r.torch = torch
        r.g = g
        r.plan = dist.slab_decompose(g, syms, P)
        r.rank = rank
        r.lg = r.plan.local_graph(rank)
        r.ex = GpuExecutor(r.lg, syms, device=0, options=InterpOptions(), dynamic_p0=True)
        r.nccl = _NoTransfer()
        r.xchg = dist.HaloExchanger(r.plan, rank, r._rows_of, transport=r._transport)
        r.ex.op_hook = r._hook
        r._exchanged = set()
        r.force_split = False
        r.splits = 0
        L = rt.lib()
        a, b, c = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        rt.check(L.b2_stream_create(ctypes.byref(a))); rt.check(L.b2_event_create(ctypes.byref(b)))
        rt.check(L.b2_event_create(ctypes.byref(c)))
        r.side, r.ev_fork, r.ev_join = a.value, b.value, c.value
        r.ex.map_split = r._split
        r.load_inputs(inputs)
        t = time_runner(r)
        worst = max(worst, t)
        print(json.dumps({"P": P, "rank": rank, "ms_per_run": t, "splits": r.splits,
                          "launches": getattr(r.ex, "trace_launches", None)}), flush=True)
        r.ex.close()
    res[P] = {"ms": worst, "efficiency": t1 / (P * worst)}
    print(json.dumps({"P": P, "worst_rank_ms": worst, "projected_efficiency": t1 / (P * worst)}),
          flush=True)
json.dump(res, open("gpurun_out/scaling_projection.json", "w"), indent=1)
