"""The numpy / C restatements of the reference CPU path (oracle/kernels_np,
oracle/c) are pinned bitwise to evaluate_program outputs of the reference
(golden vectors), so they can serve as full-size oracles on the GPU box."""

import numpy as np
import pytest

from conftest import MANIFEST, load_case

from oracle import kernels_np as K


def _cases(name):
    return MANIFEST["kernels"][name]["cases"]


@pytest.mark.parametrize("case", _cases("jacobi_2d"), ids=lambda c: c["file"])
def test_jacobi_2d_ports(case):
    d, x = load_case(case)
    T = case["symbols"]["TSTEPS"]
    out = K.jacobi_2d(x["A"].copy(), x["B"].copy(), T)
    for k in out:
        assert np.array_equal(out[k], d["oracle/" + k])
    A, B = x["A"].copy(), x["B"].copy()
    K.jacobi_2d_c(A, B, T)
    assert np.array_equal(A, d["oracle/A"]) and np.array_equal(B, d["oracle/B"])


@pytest.mark.parametrize("case", _cases("heat_3d"), ids=lambda c: c["file"])
def test_heat_3d_ports(case):
    d, x = load_case(case)
    T = case["symbols"]["TSTEPS"]
    out = K.heat_3d(x["A"].copy(), x["B"].copy(), T)
    for k in out:
        assert np.array_equal(out[k], d["oracle/" + k])
    A, B = x["A"].copy(), x["B"].copy()
    K.heat_3d_c(A, B, T)
    assert np.array_equal(A, d["oracle/A"]) and np.array_equal(B, d["oracle/B"])


@pytest.mark.parametrize("name", ["gemver", "atax", "bicg", "go_fast", "azimint_naive"])
def test_other_ports(name):
    fn = getattr(K, name)
    for case in _cases(name):
        d, x = load_case(case)
        params = MANIFEST["kernels"][name]["params"]
        args = [x[p].copy() if x[p].ndim else float(x[p]) for p in params if p in x]
        out = fn(*args)
        for k, v in out.items():
            ref = d["oracle/" + k]
            if name in ("go_fast", "azimint_naive"):
                assert np.array_equal(v, ref, equal_nan=True), (name, k)
            else:  # BLAS: same library as the reference run here
                assert np.allclose(v, ref, rtol=1e-13, atol=1e-13), (name, k)


@pytest.mark.parametrize("name", ["conv2d_bias", "nbody", "softmax"])
def test_sweep_ports(name):
    fn = getattr(K, name)
    ent = MANIFEST["kernels"][name]
    for case in ent["cases"]:
        d, x = load_case(case)
        params = ent["params"]
        args = []
        for p in params:
            if p in x:
                args.append(x[p].copy() if x[p].ndim else float(x[p]))
            else:
                args.append(case["symbols"][p])
        out = fn(*args)
        for k, v in out.items():
            ref = d["oracle/" + k]
            if name in ("softmax", "nbody"):  # vectorised exp/pow vs scalar calls: <= 1 ulp
                assert np.allclose(v, ref, rtol=1e-14, atol=0), (name, k)
            else:
                assert np.array_equal(v, ref, equal_nan=True), (name, k, np.abs(v - ref).max())


def test_threaded_cpu_ports_bitwise():
    """The reference-arm ports split planes over host threads: same
    per-element op order, so bitwise equal to the serial restatement."""
    import numpy as np

    from oracle import kernels_np as K

    rng = np.random.default_rng(11)
    A = rng.uniform(-1, 1, (37, 30, 29))
    B = rng.uniform(-1, 1, (37, 30, 29))
    A2, B2 = A.copy(), B.copy()
    K.heat_3d_sweeps(A, B, 5)
    K.heat_3d_sweeps_mt(A2, B2, 5, 6)
    assert np.array_equal(A, A2) and np.array_equal(B, B2)
    A = rng.uniform(-1, 1, (101, 77))
    B = rng.uniform(-1, 1, (101, 77))
    A2, B2 = A.copy(), B.copy()
    K.jacobi_2d(A, B, 4)  # 3 iterations = 6 sweeps
    K.jacobi_2d_sweeps_mt(A2, B2, 6, 4)
    assert np.array_equal(A, A2) and np.array_equal(B, B2)
