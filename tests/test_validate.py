"""The validator restatement (validate.py) against the reference's own
``Sdfg.validate`` (pkg/src/sdfgkit/ir.py:595-745): identical error-code sets
on the reference-generated validation fixtures and on every golden graph;
``interpret`` refuses a graph with an error diagnostic unless
``skip_validation`` is set (interp.py:184-189)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN

CASES = json.loads((GOLDEN / "validation_cases.json").read_text())


@pytest.mark.parametrize("name", sorted(CASES))
def test_validator_matches_reference(name):
    from paper_2107_00555_b200 import sdfg, validate

    case = CASES[name]
    ours = sorted({d.code for d in validate.errors(sdfg.from_dict(case["graph"]))})
    assert ours == case["reference_error_codes"]


def test_golden_graphs_validate_clean():
    from paper_2107_00555_b200 import sdfg, validate

    for p in sorted((GOLDEN / "graphs").glob("*.json")):
        assert validate.errors(sdfg.load(p)) == [], p.name


@pytest.mark.parametrize("name", ["race_whole", "map_conflict", "inplace_neighbour",
                                  "unprovable_two_syms"])
def test_interpret_rejects_racy_graph(name):
    """Raised before any device work, so this runs without a GPU."""
    from paper_2107_00555_b200 import ExecContext, InterpreterError, interpret

    g = CASES[name]["graph"]
    ctx = ExecContext(bindings={"N": 8, "M": 8}).bind_inputs(
        {"A": np.zeros(8), "x": 1.0, "B": np.zeros(8)})
    with pytest.raises(InterpreterError, match="graph does not validate: .*data race"):
        interpret(g, ctx)


def test_symbolic_disjointness_rules():
    """symbolic.py:639-678 on hand cases: interval separation, congruence,
    provable overlap, unknown."""
    from paper_2107_00555_b200 import symexpr, validate as V

    def dim(t):
        return symexpr.parse_subset(t)[0]

    lo = {"N": 1}
    assert V.dim_disjoint(dim("0:N - 2:1"), dim("N - 1:N - 1:1"), lo) == V.TRUE
    assert V.dim_disjoint(dim("0:N - 1:2"), dim("1:N - 1:2"), lo) == V.TRUE
    assert V.dim_disjoint(dim("0:N - 1:1"), dim("0:N - 1:1"), lo) == V.FALSE
    assert V.dim_disjoint(dim("0:M - 1:1"), dim("N - 1:N - 1:1"), {"N": 1, "M": 1}) == V.UNKNOWN
    assert V.dim_disjoint(dim("0:3:1"), dim("4:7:1"), lo) == V.TRUE
