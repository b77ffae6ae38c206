#!/usr/bin/env python
"""Benchmark: BASELINE.json's metric ("NPBench kernel time & HBM GB/s vs
roofline; 1/2/4/8-GPU scaling efficiency") on the B200 backend.

Default workload: heat_3d float64 N=400 TSTEPS=100 (BASELINE.json configs[2]
— the config quoted both on 1 GPU and slab-decomposed over 2/4/8 GPUs, so one
workload carries the whole 1/2/4/8 scaling curve).  One step = one complete
program run (99 iterations x 2 fused 7-point sweeps) through the executor.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload heat_3d|jacobi_2d]

``value`` = algorithmic HBM bytes of the whole run / device time, inputs
resident in HBM; ``e2e`` = the same metric through the public
``interpret(g, ctx)`` with pinned host inputs, H2D + D2H inside the timed
region.  ``--impl reference`` times the reference's own CPU path (the
unmodified ``sdfgkit.frontend.evaluate_program`` installed under
baseline/_ref) on a bounded sample of the same config (2 sweeps).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import pathlib
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def _heat_bytes(N):  # per sweep: read A (N^3) + write B interior ((N-2)^3), f64
    return 8 * N ** 3 + 8 * (N - 2) ** 3


def _jac_bytes(N):
    return 8 * N ** 2 + 8 * (N - 2) ** 2


WORKLOADS = {
    "heat_3d": {
        "graph": "heat_3d.raw", "syms": {"N": 400, "TSTEPS": 100},
        "desc": "heat_3d float64 N=400 TSTEPS=100 (BASELINE configs[2])",
        "sweeps": lambda s: 2 * (s["TSTEPS"] - 1), "sweep_bytes": lambda s: _heat_bytes(s["N"]),
        "points": lambda s: (s["N"] - 2) ** 3,
        "l2_note": "inputs (2 x N^3 f64 = 1 GB) larger than the 126 MB L2; no flush",
    },
    "jacobi_2d": {
        "graph": "jacobi_2d.raw", "syms": {"N": 2000, "TSTEPS": 100},
        "desc": "jacobi_2d float64 N=2000 TSTEPS=100 (BASELINE configs[0])",
        "sweeps": lambda s: 2 * (s["TSTEPS"] - 1), "sweep_bytes": lambda s: _jac_bytes(s["N"]),
        "points": lambda s: (s["N"] - 2) ** 2,
        "l2_resident": True,
        "l2_note": "2 x 32 MB inputs fit in L2: 256 MB memset between timed steps "
                   "(outside the per-step events); within a run the sweeps are L2-resident",
    },
}


FLUSH_BYTES = 256 << 20


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons streamed (every 50 ms) during the
    timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.samples = []
        self.gpu = gpu_index
        self.proc = None
        self.t = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.strip().split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the timed region starts only once the sampler is streaming
            t0 = time.time()
            while not self.samples and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.samples.clear()
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.06)  # at least one sample even for short regions
            self.proc.terminate()  # our own child, by handle
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self.t is not None:
                self.t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def make_inputs(g, syms, seed=0):
    """make_inputs semantics of the reference conftest (pkg/tests/conftest.py:
    38-49): arrays uniform(-1, 1), f64 scalars uniform(0.5, 1.5)."""
    from paper_2107_00555_b200 import symexpr

    rng = np.random.default_rng(seed)
    out = {}
    for n, c in g.containers.items():
        if c.transient:
            continue
        shape = tuple(symexpr.evaluate(d, syms) for d in c.shape)
        out[n] = rng.uniform(-1.0, 1.0, size=shape) if shape else np.float64(rng.uniform(0.5, 1.5))
    return out


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_sample(workload, syms, sweeps=2):
    """The reference's CPU path (numpy port of evaluate_program) on a bounded
    sample: ``sweeps`` half-steps at the full config size, the planes split
    over every host thread (same per-element op order).  Returns (GB/s
    algorithmic, seconds, description, threads)."""
    from oracle import kernels_np as K

    N = syms["N"]
    th = cpu_threads()
    rng = np.random.default_rng(0)
    if workload == "heat_3d":
        A = rng.uniform(-1, 1, (N, N, N))
        B = rng.uniform(-1, 1, (N, N, N))
        t = time.perf_counter()
        K.heat_3d_sweeps_mt(A, B, sweeps, th)
        dt = time.perf_counter() - t
        byts = sweeps * _heat_bytes(N)
    else:
        A = rng.uniform(-1, 1, (N, N))
        B = rng.uniform(-1, 1, (N, N))
        t = time.perf_counter()
        K.jacobi_2d_sweeps_mt(A, B, sweeps, th)
        dt = time.perf_counter() - t
        byts = sweeps * _jac_bytes(N)
    return (byts / dt / 1e9, dt, f"{sweeps} sweeps of {workload} N={N} via numpy "
            f"(evaluate_program port, planes split over {th} threads)", th)


REF_DIR = ROOT / "baseline" / "_ref"


def reference_sample(workload, syms):
    """The UNMODIFIED reference's own CPU path on a bounded sample: the
    reference package installed under baseline/_ref (pip --target, see
    DESIGN.md), ``sdfgkit.frontend.evaluate_program`` (pkg/src/sdfgkit/
    frontend/oracle.py:37-70) on the same DSL program at the full config size
    with TSTEPS=2 (exactly 2 sweeps; one evaluate_program call, input copies
    included as the reference makes them).  Returns (GB/s algorithmic,
    seconds, description, threads) or None when the package is absent."""
    if not (REF_DIR / "sdfgkit").is_dir():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    from sdfgkit import frontend

    prog_file = {"heat_3d": ROOT / "programs" / "heat_3d.dpy"}.get(workload)
    if prog_file is None:  # the reference corpus program (copied there by build())
        prog_file = REF_DIR / "corpus" / f"{workload}.dpy"
        if not prog_file.exists():
            return None
    program = frontend.parse(prog_file.read_text())
    N = syms["N"]
    s2 = dict(syms, TSTEPS=2)
    rng = np.random.default_rng(0)
    shape = (N, N, N) if workload == "heat_3d" else (N, N)
    inputs = {"A": rng.uniform(-1, 1, shape), "B": rng.uniform(-1, 1, shape)}
    t = time.perf_counter()
    frontend.evaluate_program(program, s2, inputs)
    dt = time.perf_counter() - t
    byts = 2 * (_heat_bytes(N) if workload == "heat_3d" else _jac_bytes(N))
    blas = os.environ.get("OPENBLAS_NUM_THREADS", "unset")
    return (byts / dt / 1e9, dt,
            f"reference sdfgkit.frontend.evaluate_program (baseline/_ref, unmodified) on "
            f"{prog_file.name} N={N} TSTEPS=2 = 2 sweeps; numpy elementwise ops are "
            f"single-threaded (OPENBLAS_NUM_THREADS={blas}, unused here)", 1)


def run_reference(args, W):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    syms = W["syms"]
    kind = "reference"
    sample = lambda: reference_sample(args.workload, syms)  # noqa: E731
    if sample() is None:  # not installed: the numpy port (kind "port")
        kind = "port"
        sample = lambda: cpu_sample(args.workload, syms, 2)  # noqa: E731
    for _ in range(max(0, args.warmup - 1)):
        sample()
    vals, ts = [], []
    for _ in range(args.steps):
        v, dt, desc, th = sample()
        vals.append(v)
        ts.append(dt)
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": metric_name(args.workload), "value": value,
        "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.median(ts)), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": W["desc"], "sample": desc},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": th, "kind": kind,
                         "sample": desc},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name(workload):
    return f"{workload}_f64_algorithmic_hbm_GBps"


def traffic_from_profiles(workload):
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    w = d.get(workload)
    return None if w is None else w.get("dram_bytes_per_launch")


def run_ours(args, W):
    from paper_2107_00555_b200 import ExecContext, InterpOptions, interpret, runtime as rt, sdfg
    from paper_2107_00555_b200.machine import get_executor

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1 or os.environ.get("B2_FORCE_SLAB"):
        from paper_2107_00555_b200.dist import bench_slab
        return bench_slab(args, W)

    syms = W["syms"]
    g = sdfg.load(ROOT / "tests" / "golden" / "graphs" / f"{W['graph']}.json")
    inputs = make_inputs(g, syms)
    ex = get_executor(g, syms)
    L = rt.lib()
    ex.prepare_inputs(inputs)
    ex.sync()
    run_bytes = W["sweeps"](syms) * W["sweep_bytes"](syms)

    # warm-up (first call traces the state machine and captures the CUDA graph)
    for i in range(args.warmup):
        ex.run_device(first_call=(i == 0))
    ex.sync()
    launches_per_step = getattr(ex, "trace_launches", None)

    # one event pair per step; when the working set fits in L2 (jacobi_2d's
    # 2 x 32 MB) a 256 MB memset between steps evicts it, outside the events
    flush = W.get("l2_resident", False)
    fbuf = ctypes.c_void_p()
    if flush:
        rt.check(L.b2_malloc(ctypes.byref(fbuf), FLUSH_BYTES))
    evs = []
    for _ in range(args.steps):
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        L.b2_event_create(ctypes.byref(a))
        L.b2_event_create(ctypes.byref(b))
        evs.append((a, b))
    with ClockSampler() as clk:
        ex.sync()
        for a, b in evs:
            if flush:
                rt.check(L.b2_memset(fbuf, 0, FLUSH_BYTES, ex.stream))
            L.b2_event_record(a, ex.stream)
            ex.run_device(first_call=False)
            L.b2_event_record(b, ex.stream)
        ex.sync()
    tot_ms = 0.0
    for a, b in evs:
        ms = ctypes.c_float()
        rt.check(L.b2_event_elapsed_ms(a, b, ctypes.byref(ms)))
        tot_ms += ms.value
    ms_per_step = tot_ms / args.steps
    if flush:
        L.b2_free(fbuf)
    value = run_bytes / (ms_per_step / 1e3) / 1e9
    ex.check_flag()

    # dominant kernel: per-launch CUDA events on the launching stream
    prof = ex.profile_launches()
    name, (nl, tot, npts) = max(prof.items(), key=lambda kv: kv[1][1])
    avg_ms = tot / nl
    kern_ms = sum(t for (_, t, _) in prof.values())
    time_basis = "CUDA-event pairs around every launch, captured and replayed as one graph"
    if kern_ms > ms_per_step:
        # the pairs break programmatic-dependent-launch overlap and add a gap
        # per launch, inflating short kernels: take the kernel's event-pair
        # share of the plain step instead
        avg_ms = ms_per_step * tot / kern_ms / nl
        time_basis += "; scaled to the plain step (the kernels' sum exceeded it)"
    per_launch = W["sweep_bytes"](syms)
    peak, peak_kind = peaks()
    achieved = per_launch / (avg_ms / 1e3) / 1e9
    step_share = tot / max(ms_per_step, kern_ms)
    # the program alternates two sweep kernels with the same body (B = f(A),
    # A = f(B)): their combined share of the step
    family = [k for k, (_, _, p) in prof.items() if p == npts]
    family_share = sum(prof[k][1] for k in family) / max(ms_per_step, kern_ms)

    # end to end through the public API: pinned host inputs, H2D + D2H timed
    host = {k: np.ascontiguousarray(v) for k, v in inputs.items()}
    for v in host.values():
        if v.nbytes:
            L.b2_host_register(v.ctypes.data, v.nbytes)
    ctx = ExecContext(bindings=dict(syms))
    ctx.bind_inputs(host)
    opts = InterpOptions(pinned_outputs=True)  # page-locked D2H staging
    interpret(g, ctx, opts)  # warm
    t = time.perf_counter()
    for _ in range(args.steps):
        out = interpret(g, ctx, opts)
    e2e_s = (time.perf_counter() - t) / args.steps
    # bytes actually moved host -> device (inputs whose interior is dead on
    # entry upload only their boundary faces, machine._dead_on_entry)
    h2d = getattr(ex, "last_h2d_bytes", None) or sum(v.nbytes for v in host.values())
    d2h = sum(np.asarray(v).nbytes for v in out.values())

    port_v, port_dt, port_desc, port_th = cpu_sample(args.workload, syms, 2)
    refs = reference_sample(args.workload, syms)
    if refs is not None:
        cpu_v, cpu_dt, cpu_desc, cpu_th = refs
        cpu_kind = "reference"
    else:
        cpu_v, cpu_dt, cpu_desc, cpu_th, cpu_kind = port_v, port_dt, port_desc, port_th, "port"

    line = {
        "metric": metric_name(args.workload), "value": value, "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (make_inputs semantics, seed 0)",
        "config": {"workload": W["desc"], "graph": f"tests/golden/graphs/{W['graph']}.json",
                   "l2": W["l2_note"],
                   "algorithmic_bytes_per_step": run_bytes},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind,
                     "traffic": traffic_from_profiles(args.workload), "kernel": name,
                     "launch_ms": avg_ms, "launch_time_basis": time_basis,
                     "launches_per_step": nl, "step_share": step_share,
                     "sweep_kernels": sorted(family), "sweep_share": family_share,
                     "bytes_per_launch": per_launch},
        "cpu_baseline": {"value": cpu_v, "unit": "GB/s", "cores": cpu_th, "kind": cpu_kind,
                         "sample": cpu_desc, "seconds": cpu_dt},
        "cpu_baseline_port": {"value": port_v, "unit": "GB/s", "cores": port_th, "kind": "port",
                              "sample": port_desc, "seconds": port_dt},
        "e2e": {"value": run_bytes / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3},
        "gpu_launches": (launches_per_step or nl) * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="heat_3d",
                    choices=sorted(WORKLOADS) + ["matmul", "matmul_f32", "jacobi_2d_local"])
    ap.add_argument("--n", type=int, default=16384, help="SUMMA size (matmul workloads)")
    args = ap.parse_args()
    if args.workload.startswith("matmul"):
        if args.impl == "reference":
            rank = int(os.environ.get("RANK", "0"))
            if rank == 0:
                from oracle import kernels_np as K
                n = 4096
                rng = np.random.default_rng(0)
                A, B = rng.uniform(-1, 1, (n, n)), rng.uniform(-1, 1, (n, n))
                t = time.perf_counter()
                K.matmul(A, B)
                dt = time.perf_counter() - t
                v = 2 * n ** 3 / dt / 1e12
                print(json.dumps({"impl": "reference", "metric": f"summa_{args.workload}_TFLOPs",
                                  "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
                                  "cpu_baseline": {"value": v, "unit": "TFLOP/s", "kind": "port",
                                                   "cores": os.cpu_count(),
                                                   "sample": "4096^3 numpy/OpenBLAS dgemm"},
                                  "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}), flush=True)
            return
        from paper_2107_00555_b200.dist import bench_summa
        return bench_summa(args, args.n, "f32" if args.workload.endswith("f32") else "f64")
    if args.workload == "jacobi_2d_local":
        W = WORKLOADS["jacobi_2d"]
        if args.impl == "reference":
            args.workload = "jacobi_2d"
            return run_reference(args, W)
        from paper_2107_00555_b200.comm import bench_local_view
        return bench_local_view(args, W)
    W = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, W)
    else:
        run_ours(args, W)


if __name__ == "__main__":
    main()
