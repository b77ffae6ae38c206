"""GPU parity: the B200 executor against the reference's own outputs.

For every golden kernel (reference corpus + repo programs), every graph
variant (raw / pipe / auto) and every size/seed case, ``interpret`` on the
B200 must match the reference interpreter run on the SAME graph variant
(tests/golden, produced by make_golden.py from /root/reference):
  * bitwise for kernels whose op order is fixed by the tasklet chain
    (stencils, elementwise, scalar code) — the reference's own oracle-suite
    criterion (pkg/tests/test_oracle_suite.py:47-48),
  * within rel_err 1e-12 (north-star float64 tolerance) where the device
    re-associates sums (WCR reductions, matmul, reduce).
"""

import numpy as np
import pytest

from conftest import golden_cases, load_case, rel_err

pytestmark = pytest.mark.gpu

BITWISE = {"jacobi_1d", "jacobi_2d", "heat_3d", "fig4_loop", "adi"}
TOL = 1e-12


def _run(name, variant, case):
    from paper_2107_00555_b200 import ExecContext, interpret, sdfg
    from conftest import GOLDEN

    g = sdfg.load(GOLDEN / "graphs" / f"{name}.{variant}.json")
    d, inputs = load_case(case)
    ctx = ExecContext(bindings=dict(case["symbols"]))
    ctx.bind_inputs({k: v.copy() for k, v in inputs.items()})
    out = interpret(g, ctx)
    return out, d, ctx


@pytest.mark.parametrize("name,variant,case", golden_cases(),
                         ids=lambda x: x if isinstance(x, str) else x.get("file", ""))
def test_matches_reference_interpreter(name, variant, case):
    d0, _ = load_case(case)
    key = f"interp_{variant}/"
    bad = [k for k in d0.files if k.startswith(key)
           and rel_err(d0[k], d0["oracle/" + k[len(key):]]) > 1e-9]
    if bad:
        # the reference's own passes miscompile this variant (its interpreter
        # disagrees with its oracle, e.g. softmax after LoopToMap): the graph
        # is racy, so there is no well-defined result to match
        pytest.skip(f"reference {variant} graph disagrees with its own oracle: {bad}")
    out, d, ctx = _run(name, variant, case)
    refs = {k[len(key):]: d[k] for k in d.files if k.startswith(key)}
    assert refs, "no reference output stored for this variant"
    for k, ref in refs.items():
        err = rel_err(out[k], ref)
        assert err <= TOL, f"{name}.{variant} {case['file']} {k}: rel_err {err:.3e}"
        if name in BITWISE:
            assert np.array_equal(out[k], ref, equal_nan=True), \
                f"{name}.{variant} {k}: not bitwise equal (rel_err {err:.3e})"


@pytest.mark.parametrize("name,variant,case", [c for c in golden_cases(1) if c[1] == "raw"],
                         ids=lambda x: x if isinstance(x, str) else x.get("file", ""))
def test_matches_big_step_oracle(name, variant, case):
    """Raw graphs agree with the reference's independent AST oracle
    evaluate_program (frontend/oracle.py:37-70)."""
    out, d, _ = _run(name, variant, case)
    for k in [f[7:] for f in d.files if f.startswith("oracle/")]:
        assert rel_err(out[k], d["oracle/" + k]) <= TOL


@pytest.mark.parametrize("name,variant,case", [c for c in golden_cases(1) if c[1] == "raw"],
                         ids=lambda x: x if isinstance(x, str) else x.get("file", ""))
def test_counters_match_reference(name, variant, case):
    """map_iterations and wcr_commits restate Counters (interp.py:73-92)."""
    _, d, ctx = _run(name, variant, case)
    ref = case["counters"]["raw"]
    assert ctx.counters.map_iterations == ref["map_iterations"]
    assert ctx.counters.wcr_commits == ref["wcr_commits"]
