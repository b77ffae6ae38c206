"""Degenerate sizes (tests/golden/edges, made by make_edge_cases.py from the
reference interpreter and oracle): empty stencil interiors, loops that never
iterate, single-element / rank-1 matrices, one particle, one bin.

* CPU: the oracle restatement (oracle/interp_ref.py) equals the reference
  interpreter bitwise on every case (it is the checker, so it is pinned).
* GPU: ``interpret`` on the B200 equals the reference interpreter — bitwise
  where the op order is fixed (stencils, elementwise, scalar code), within
  rel_err 1e-12 elsewhere (re-associated sums)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, rel_err

EDGES = GOLDEN / "edges"
BITWISE = {"jacobi_1d", "jacobi_2d", "heat_3d", "fig4_loop", "go_fast"}


def _cases():
    man = json.loads((EDGES / "manifest.json").read_text())
    return [(name, c) for name, cs in sorted(man.items()) for c in cs]


def _load(name, case):
    from paper_2107_00555_b200 import sdfg

    d = np.load(EDGES / case["file"])
    ins = {k[3:]: d[k] for k in d.files if k.startswith("in/")}
    ref = {k[7:]: d[k] for k in d.files if k.startswith("interp/")}
    g = sdfg.load(GOLDEN / "graphs" / f"{name}.raw.json")
    return g, ins, ref


def _inputs(ins):
    return {k: (v.copy() if v.ndim else float(v)) for k, v in ins.items()}


@pytest.mark.parametrize("name,case", _cases(), ids=lambda x: x if isinstance(x, str)
                         else x["file"])
def test_oracle_matches_reference_on_edges(name, case):
    from oracle import interp_ref

    assert "reference_error" not in case
    g, ins, ref = _load(name, case)
    out = interp_ref.interpret(g, dict(case["symbols"]), _inputs(ins))
    for k, v in ref.items():
        assert np.array_equal(np.asarray(out[k]), v, equal_nan=True), (name, k)


@pytest.mark.gpu
@pytest.mark.parametrize("name,case", _cases(), ids=lambda x: x if isinstance(x, str)
                         else x["file"])
def test_device_matches_reference_on_edges(name, case):
    from paper_2107_00555_b200 import ExecContext, interpret

    g, ins, ref = _load(name, case)
    ctx = ExecContext(bindings=dict(case["symbols"])).bind_inputs(_inputs(ins))
    out = interpret(g, ctx)
    for k, v in ref.items():
        assert rel_err(out[k], v) <= 1e-12, (name, case["symbols"], k, rel_err(out[k], v))
        if name in BITWISE:
            assert np.array_equal(np.asarray(out[k]), v, equal_nan=True), (name, k)
