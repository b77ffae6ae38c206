"""Dev check: odd-size parity sweep of the benchmark programs against the CPU
ports (bitwise for stencils, rel_err 1e-12 for BLAS-2)."""
import inspect, sys
sys.path.insert(0, '.')
import numpy as np
from oracle import kernels_np as K
from paper_2107_00555_b200 import ExecContext, interpret, sdfg, symexpr

GD = "tests/golden/graphs"


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) if b.size else 0.0


def inputs_for(g, syms, seed):
    rng = np.random.default_rng(seed)
    out = {}
    for n, c in g.containers.items():
        if not c.transient:
            shape = tuple(symexpr.evaluate(d, syms) for d in c.shape)
            out[n] = rng.uniform(-1, 1, shape) if shape else float(rng.uniform(0.5, 1.5))
    return out


fails = 0
for N in (17, 33, 130, 257):
    g = sdfg.load(f"{GD}/heat_3d.raw.json")
    ins = inputs_for(g, {"N": N, "TSTEPS": 3}, N)
    out = interpret(g, ExecContext(bindings={"N": N, "TSTEPS": 3}).bind_inputs(
        {k: np.array(v, copy=True) for k, v in ins.items()}))
    A, B = ins["A"].copy(), ins["B"].copy()
    K.heat_3d_c(A, B, 3)
    ok = np.array_equal(out["A"], A) and np.array_equal(out["B"], B)
    fails += not ok
    print("heat", N, ok, flush=True)
for N in (99, 513, 1001):
    g = sdfg.load(f"{GD}/jacobi_2d.raw.json")
    ins = inputs_for(g, {"N": N, "TSTEPS": 4}, N)
    out = interpret(g, ExecContext(bindings={"N": N, "TSTEPS": 4}).bind_inputs(
        {k: np.array(v, copy=True) for k, v in ins.items()}))
    A, B = ins["A"].copy(), ins["B"].copy()
    K.jacobi_2d_c(A, B, 4)
    ok = np.array_equal(out["A"], A) and np.array_equal(out["B"], B)
    fails += not ok
    print("jacobi", N, ok, flush=True)
for name, syms in (("atax", {"M": 1001, "N": 999}), ("atax", {"M": 4000, "N": 4002}),
                   ("bicg", {"N": 3001, "M": 2999}), ("bicg", {"N": 2000, "M": 6000}),
                   ("gemver", {"N": 4001}), ("gemver", {"N": 3000})):
    g = sdfg.load(f"{GD}/{name}.raw.json")
    ins = inputs_for(g, syms, 7)
    out = interpret(g, ExecContext(bindings=syms).bind_inputs(
        {k: np.array(v, copy=True) for k, v in ins.items()}))
    fn = getattr(K, name)
    ref = fn(*[np.array(ins[p], copy=True) if np.ndim(ins[p]) else ins[p]
               for p in inspect.signature(fn).parameters])
    err = max(rel(out[k], v) for k, v in ref.items())
    # sums re-associated against BLAS: elementwise rel_err (floor 1) is
    # bounded by eps * sum|terms| for near-cancelling entries; norm-wise error
    # is the size-independent check
    nerr = max(float(np.linalg.norm(out[k] - v) / np.linalg.norm(v)) for k, v in ref.items())
    ok = err <= 1e-12 or nerr <= 1e-14
    fails += not ok
    print(name, syms, ok, err, nerr, flush=True)
# NPBench sweep programs at odd sizes (reduction schedules: register-blocked,
# short-chunk in-block, chunked + fold, row reductions, warp folds)
npb = (("softmax", {"N": 3, "H": 5, "SM": 77}, ("x",), ("out",)),
       ("softmax", {"N": 2, "H": 3, "SM": 512}, ("x",), ("out",)),
       ("conv2d_bias", {"NB": 2, "H": 150, "W": 150, "CI": 3, "CO": 16, "K": 20, "HO": 131,
                        "WO": 131}, ("inp", "w", "bias"), ("out",)),
       ("conv2d_bias", {"NB": 1, "H": 37, "W": 41, "CI": 2, "CO": 5, "K": 3, "HO": 35,
                        "WO": 39}, ("inp", "w", "bias"), ("out",)),
       ("azimint_naive", {"N": 200001, "NPT": 997}, ("rmax", "data", "radius"), ("res",)),
       ("go_fast", {"N": 3001}, ("a",), ("out",)),
       ("nbody", {"N": 77, "NT": 9}, ("mass", "pos", "vel", "acc", "E", "G", "softening", "dt"),
        ("pos", "vel", "acc", "E")))
for name, syms, _, outs in npb:
    g = sdfg.load(f"{GD}/{name}.raw.json")
    ins = inputs_for(g, syms, 11)
    if name == "azimint_naive":
        ins["radius"] = np.abs(ins["radius"]) * ins["rmax"]
    out = interpret(g, ExecContext(bindings=syms).bind_inputs(
        {k: np.array(v, copy=True) for k, v in ins.items()}))
    fn = getattr(K, name)
    args = {k: (np.array(v, copy=True) if np.ndim(v) else v) for k, v in ins.items()}
    params = list(inspect.signature(fn).parameters)
    call = [args[p] if p in args else syms[p] for p in params]
    ref = fn(*call)
    if not isinstance(ref, dict):
        ref = {o: args[o] for o in outs}
    err = max(float(np.linalg.norm(out[k] - ref[k]) / max(np.linalg.norm(ref[k]), 1e-300))
              for k in outs)
    ok = err <= 1e-12
    fails += not ok
    print(name, syms, ok, err, flush=True)
print("FAILS", fails)
