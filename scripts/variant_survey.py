"""Device time per run of every golden kernel's graph variants (raw / pipe /
auto / b2reg) at moderately large sizes — finds performance traps in the
graphs the reference's optimiser produces (dev tool)."""
import ctypes
import json
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_2107_00555_b200 import runtime as rt, sdfg  # noqa: E402
from paper_2107_00555_b200.machine import GpuExecutor  # noqa: E402

SIZES = {
    "atax": {"M": 4000, "N": 4000}, "bicg": {"N": 4000, "M": 4000}, "mvt": {"N": 4000},
    "gesummv": {"N": 4000}, "gemver": {"N": 4000}, "gemm": {"NI": 1024, "NJ": 1024, "NK": 1024},
    "k2mm": {"NI": 800, "NJ": 900, "NK": 1000, "NL": 700},
    "k3mm": {"NI": 600, "NJ": 700, "NK": 800, "NM": 900, "NL": 1000},
    "doitgen": {"NR": 64, "NQ": 64, "NP": 256}, "jacobi_1d": {"N": 1000000, "TSTEPS": 10},
    "jacobi_2d": {"N": 1000, "TSTEPS": 10}, "adi": {"N": 400, "TSTEPS": 5},
    "fig4_loop": {"NI": 100000}, "wcr_sum": {"NI": 2048, "NJ": 2048},
    "go_fast": {"N": 4000}, "softmax": {"N": 4, "H": 4, "SM": 256},
    "azimint_naive": {"N": 100000, "NPT": 100}, "matmul": {"M": 1024, "K": 1024, "N": 1024},
    "conv2d_bias": {"NB": 2, "H": 64, "W": 64, "CI": 3, "CO": 16, "K": 5, "HO": 60, "WO": 60},
    "nbody": {"N": 100, "NT": 10}, "heat_3d": {"N": 100, "TSTEPS": 5},
}
only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
L = rt.lib()
e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
L.b2_event_create(ctypes.byref(e0))
L.b2_event_create(ctypes.byref(e1))
for name, syms in SIZES.items():
    if only and name not in only:
        continue
    row = {}
    for v in ("raw", "pipe", "auto", "b2reg"):
        try:
            g = sdfg.load(f"tests/golden/graphs/{name}.{v}.json")
        except FileNotFoundError:
            continue
        try:
            ex = GpuExecutor(g, syms)
            rng = np.random.default_rng(0)
            ins = {}
            for n, c in g.containers.items():
                if not c.transient:
                    shp = ex.buf.shape[n]
                    ins[n] = rng.uniform(-1, 1, shp) if shp else np.float64(rng.uniform(0.5, 1.5))
            ex.prepare_inputs(ins)
            ex.sync()
            ex.run_device(first_call=True)
            ex.sync()
            ts = []
            for _ in range(3):
                L.b2_event_record(e0, ex.stream)
                ex.run_device(first_call=False)
                L.b2_event_record(e1, ex.stream)
                ms = ctypes.c_float()
                rt.check(L.b2_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
                ts.append(ms.value)
            modes = sorted({sp.mode for sp in ex.specs.values()})
            row[v] = (round(float(np.median(ts)), 3), modes)
            ex.close()
        except Exception as exn:  # noqa: BLE001
            row[v] = ("ERR", str(exn)[:80])
    print(json.dumps({"kernel": name, **{k: v for k, v in row.items()}}), flush=True)
