"""CPU ORACLE — test infrastructure only (tests/, smoke(), bench.py's CPU
baseline leg); never the product path.

numpy restatements of the reference's CPU path for the benchmark programs,
i.e. what ``sdfgkit.frontend.evaluate_program`` (pkg/src/sdfgkit/frontend/
oracle.py:37-70) does on them: every slice statement evaluated as
whole-array numpy binary ops, left to right (eval_expr, oracle.py:205-262),
then assigned (exec_assign, oracle.py:126-156); ``@`` is numpy/BLAS
(oracle.py:238); explicit ``map[...]`` bodies run per element (oracle.py:
116-124) — restated here vectorised with the same per-element op order.
These reproduce evaluate_program bitwise (pinned by tests against the golden
vectors from the reference) and run at BASELINE.json's config sizes.

Programs: jacobi_2d / gemver / atax / bicg are the reference corpus
(pkg/tests/corpus/*.dpy); heat_3d and the NPBench-sweep kernels are this
repo's DSL programs (programs/*.dpy).
"""

from __future__ import annotations

import ctypes
import math
import os
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent


def jacobi_2d(A, B, TSTEPS):
    for _t in range(1, TSTEPS):
        B[1:-1, 1:-1] = 0.2 * (A[1:-1, 1:-1] + A[1:-1, :-2] + A[1:-1, 2:] + A[2:, 1:-1] + A[:-2, 1:-1])
        A[1:-1, 1:-1] = 0.2 * (B[1:-1, 1:-1] + B[1:-1, :-2] + B[1:-1, 2:] + B[2:, 1:-1] + B[:-2, 1:-1])
    return {"A": A, "B": B}


def _heat_rhs(A):
    return (0.125 * (A[2:, 1:-1, 1:-1] - 2.0 * A[1:-1, 1:-1, 1:-1] + A[:-2, 1:-1, 1:-1])
            + 0.125 * (A[1:-1, 2:, 1:-1] - 2.0 * A[1:-1, 1:-1, 1:-1] + A[1:-1, :-2, 1:-1])
            + 0.125 * (A[1:-1, 1:-1, 2:] - 2.0 * A[1:-1, 1:-1, 1:-1] + A[1:-1, 1:-1, 0:-2])
            + A[1:-1, 1:-1, 1:-1])


def heat_3d(A, B, TSTEPS):
    for _t in range(1, TSTEPS):
        B[1:-1, 1:-1, 1:-1] = _heat_rhs(A)
        A[1:-1, 1:-1, 1:-1] = _heat_rhs(B)
    return {"A": A, "B": B}


def heat_3d_sweeps(A, B, sweeps):
    """``sweeps`` half-steps (bounded CPU-baseline sample)."""
    for s in range(sweeps):
        if s % 2 == 0:
            B[1:-1, 1:-1, 1:-1] = _heat_rhs(A)
        else:
            A[1:-1, 1:-1, 1:-1] = _heat_rhs(B)


def _slabs(n_planes, threads):
    """Interior planes 1..n-2 split into contiguous [lo, hi) chunks."""
    lo, hi = 1, n_planes - 1
    k = max(1, min(threads, hi - lo))
    return [(lo + (hi - lo) * i // k, lo + (hi - lo) * (i + 1) // k) for i in range(k)]


def heat_3d_sweeps_mt(A, B, sweeps, threads):
    """heat_3d_sweeps on ``threads`` host threads: each thread evaluates the
    same whole-slice expression on a contiguous slab of planes (numpy releases
    the GIL), so every element sees the same op order — bitwise equal."""
    from concurrent.futures import ThreadPoolExecutor

    parts = _slabs(A.shape[0], threads)
    with ThreadPoolExecutor(len(parts)) as pool:
        for s in range(sweeps):
            src, dst = (A, B) if s % 2 == 0 else (B, A)

            def work(b, src=src, dst=dst):
                lo, hi = b
                dst[lo:hi, 1:-1, 1:-1] = _heat_rhs(src[lo - 1:hi + 1])
            list(pool.map(work, parts))


def jacobi_2d_sweeps_mt(A, B, sweeps, threads):
    from concurrent.futures import ThreadPoolExecutor

    parts = _slabs(A.shape[0], threads)

    def rhs(X, lo, hi):
        return 0.2 * (X[lo:hi, 1:-1] + X[lo:hi, :-2] + X[lo:hi, 2:] + X[lo + 1:hi + 1, 1:-1]
                      + X[lo - 1:hi - 1, 1:-1])
    with ThreadPoolExecutor(len(parts)) as pool:
        for s in range(sweeps):
            src, dst = (A, B) if s % 2 == 0 else (B, A)

            def work(b, src=src, dst=dst):
                lo, hi = b
                dst[lo:hi, 1:-1] = rhs(src, lo, hi)
            list(pool.map(work, parts))


def gemver(alpha, beta, A, u1, v1, u2, v2, w, x, y, z):
    # explicit map: A[i, j] = A[i, j] + u1[i] * v1[j] + u2[i] * v2[j] (per element,
    # left to right: (A + u1*v1) + u2*v2)
    A[:, :] = (A + np.outer(u1, v1)) + np.outer(u2, v2)
    x[:] = x + beta * (y @ A) + z
    w[:] = alpha * (A @ x)
    return {"A": A, "x": x, "w": w}


def atax(A, x, y):
    y[:] = (A @ x) @ A
    return {"y": y}


def bicg(A, s, q, p, r):
    s[:] = r @ A
    q[:] = A @ p
    return {"s": s, "q": q}


def go_fast(a, out):
    trace = 0.0
    for i in range(a.shape[0]):
        e2 = math.exp(2.0 * a[i, i])
        trace += (e2 - 1.0) / (e2 + 1.0)
    out[:] = a + trace
    return {"out": out}


def azimint_naive(rmax, data, radius, res):
    NPT = res.shape[0]
    i = np.arange(NPT, dtype=np.float64)[:, None]
    lo = rmax * i / NPT
    hi = rmax * (i + 1) / NPT
    mask = (lo <= radius[None, :]) & (radius[None, :] < hi)
    # the map's WCR sums run lexicographically (i outer, k inner): sequential in k
    acc = np.zeros(NPT)
    cnt = np.zeros(NPT)
    for k in range(radius.shape[0]):
        acc = acc + mask[:, k] * data[k]
        cnt = cnt + mask[:, k] * 1.0
    with np.errstate(invalid="ignore", divide="ignore"):
        res[:] = acc / cnt
    return {"res": res}


def matmul(A, B):
    return A @ B


# ---------------------------------------------------------------------------
# compiled C restatement (oracle/c/stencils.c, OpenMP over planes)

_lib = None


def c_lib():
    global _lib
    if _lib is None:
        p = HERE / "liboracle.so"
        if not p.exists():
            raise FileNotFoundError(f"{p} missing: run `make -C oracle`")
        _lib = ctypes.CDLL(str(p))
        for fn in ("oracle_heat_3d", "oracle_jacobi_2d", "oracle_heat_3d_sweeps"):
            f = getattr(_lib, fn)
            f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long, ctypes.c_long,
                          ctypes.c_int]
            f.restype = None
    return _lib


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def heat_3d_c(A, B, TSTEPS, threads=0):
    assert A.flags.c_contiguous and B.flags.c_contiguous and A.dtype == np.float64
    c_lib().oracle_heat_3d(A.ctypes.data, B.ctypes.data, A.shape[0], TSTEPS, threads)
    return {"A": A, "B": B}


def heat_3d_sweeps_c(A, B, sweeps, threads=0):
    c_lib().oracle_heat_3d_sweeps(A.ctypes.data, B.ctypes.data, A.shape[0], sweeps, threads)


def jacobi_2d_c(A, B, TSTEPS, threads=0):
    assert A.flags.c_contiguous and B.flags.c_contiguous and A.dtype == np.float64
    c_lib().oracle_jacobi_2d(A.ctypes.data, B.ctypes.data, A.shape[0], TSTEPS, threads)
    return {"A": A, "B": B}


def conv2d_bias(inp, w, bias, out):
    """programs/conv2d_bias.dpy: per output element the 7-D map accumulates
    over (ki, kj, ci) in lexicographic order after the bias init."""
    NB, H, W_, CI = inp.shape
    K = w.shape[0]
    HO, WO = out.shape[1], out.shape[2]
    out[...] = bias[None, None, None, :]
    for ki in range(K):
        for kj in range(K):
            for ci in range(CI):
                out += inp[:, ki:ki + HO, kj:kj + WO, ci, None] * w[ki, kj, ci, :]
    return {"out": out}


def _get_acc(pos, mass, acc, G, softening):
    acc[...] = 0.0
    N = pos.shape[0]
    for j in range(N):  # lexicographic (i, j): per i the WCR sum runs over j in order
        dx = pos[j, 0] - pos[:, 0]
        dy = pos[j, 1] - pos[:, 1]
        dz = pos[j, 2] - pos[:, 2]
        inv = np.power(dx * dx + dy * dy + dz * dz + softening * softening, -1.5)
        acc[:, 0] += G * (dx * inv) * mass[j]
        acc[:, 1] += G * (dy * inv) * mass[j]
        acc[:, 2] += G * (dz * inv) * mass[j]


def nbody(mass, pos, vel, acc, E, G, softening, dt, NT):
    """programs/nbody.dpy (NPBench nbody, leapfrog + energies)."""
    _get_acc(pos, mass, acc, G, softening)
    for _t in range(NT):
        vel[:] = vel + acc * (dt / 2.0)
        pos[:] = pos + vel * dt
        _get_acc(pos, mass, acc, G, softening)
        vel[:] = vel + acc * (dt / 2.0)
    N = pos.shape[0]
    E[0] = 0.0
    E[1] = 0.0
    for i in range(N):
        E[0] += 0.5 * mass[i] * (vel[i, 0] * vel[i, 0] + vel[i, 1] * vel[i, 1] + vel[i, 2] * vel[i, 2])
    for i in range(N):
        dx = pos[:, 0] - pos[i, 0]
        dy = pos[:, 1] - pos[i, 1]
        dz = pos[:, 2] - pos[i, 2]
        jj = np.arange(N)
        term = -(G * mass[i] * mass) * (i < jj) / np.sqrt(dx * dx + dy * dy + dz * dz + (i == jj))
        for j in range(N):
            E[1] += term[j]
    return {"mass": mass, "pos": pos, "vel": vel, "acc": acc, "E": E}


_exp_ufunc = np.frompyfunc(math.exp, 1, 1)


def _math_exp(a):
    out = np.empty_like(a)
    flat, dst = a.reshape(-1), out.reshape(-1)
    for s in range(0, flat.size, 1 << 22):  # chunked: bounded object temporaries
        dst[s:s + (1 << 22)] = _exp_ufunc(flat[s:s + (1 << 22)]).astype(np.float64)
    return out


def softmax(x, out):
    """programs/softmax.dpy: row max by a sequential scan, exp(x - max), row
    sum by WCR in l order, divide."""
    mx = x[..., 0].copy()
    for l in range(1, x.shape[-1]):
        mx = np.maximum(mx, x[..., l]) if False else np.where(x[..., l] > mx, x[..., l], mx)
    # exp is math.exp per element in the reference (oracle.py:23, the map
    # body runs per point); numpy's vectorised exp can differ by an ulp
    ex = _math_exp(x - mx[..., None])
    sm = np.zeros(x.shape[:-1])
    for l in range(x.shape[-1]):
        sm = sm + ex[..., l]
    out[...] = ex / sm[..., None]
    return {"out": out}
