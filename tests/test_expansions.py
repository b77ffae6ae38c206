"""The b200 library plug-in (expansions.py) against the reference's own
expansion machinery (ExpansionRegistry / expand_library / auto_optimize,
pkg/src/sdfgkit/autoopt.py:640-667, 923-1004)."""

import json
import pathlib

import numpy as np
import pytest

from conftest import GOLDEN, MANIFEST, ROOT

REF_DIRS = [ROOT / "baseline" / "_ref", pathlib.Path("/root/reference/pkg/src")]


def _sdfgkit():
    import sys

    for d in REF_DIRS:
        if (d / "sdfgkit").is_dir() and str(d) not in sys.path:
            sys.path.insert(0, str(d))
    return pytest.importorskip("sdfgkit")


def _corpus(name):
    for d in (ROOT / "baseline" / "_ref" / "corpus", pathlib.Path("/root/reference/pkg/tests/corpus")):
        if (d / f"{name}.dpy").exists():
            return (d / f"{name}.dpy").read_text()
    pytest.skip("reference corpus not available")


def test_b2reg_goldens_keep_library_nodes():
    """auto_optimize with the b200 registry leaves no top-level MATMUL /
    REDUCE / TRANSPOSE (expand_library's loop condition, autoopt.py:969-981)
    and the loader puts the wrapped nodes back onto the outer memlets."""
    from paper_2107_00555_b200 import sdfg

    seen = 0
    for name, ent in MANIFEST["kernels"].items():
        if "b2reg" not in ent["variants"]:
            continue
        doc = json.loads((GOLDEN / "graphs" / f"{name}.b2reg.json").read_text())
        top = [n for st in doc["states"] for n in st["nodes"]
               if n["type"] == "library" and n["kind"] in ("matmul", "reduce", "transpose")]
        assert not top, name
        wrapped = [n for st in doc["states"] for n in st["nodes"]
                   if n["type"] == "nested" and n["sdfg"]["name"].startswith("b200_lib_")]
        g = sdfg.load(GOLDEN / "graphs" / f"{name}.b2reg.json")
        libs = [n for st in g.states for n in st.nodes if isinstance(n, sdfg.Library)]
        assert len(libs) == len(wrapped), name
        assert not any(isinstance(n, sdfg.Nested) and n.sdfg.name.startswith("b200_lib_")
                       for st in g.states for n in st.nodes)
        seen += len(wrapped)
    assert seen >= 10


@pytest.mark.parametrize("name,syms", [("atax", {"M": 6, "N": 5}), ("gemver", {"N": 6}),
                                       ("doitgen", {"NR": 3, "NQ": 4, "NP": 5}),
                                       ("k3mm", {"NI": 3, "NJ": 4, "NK": 5, "NM": 2, "NL": 3})])
def test_registry_semantics_preserved_in_reference(name, syms):
    """expand_library(g, registry=b200_registry(cpu_registry())) output runs
    in the REFERENCE interpreter bitwise equal to its oracle, validates,
    and pinning still selects the CPU expansions (autoopt.py:656-664)."""
    sk = _sdfgkit()
    from sdfgkit import autoopt, frontend
    from sdfgkit.interp import ExecContext, interpret

    from paper_2107_00555_b200 import expansions as X

    src = _corpus(name)
    prog = frontend.parse(src)
    g, _ = frontend.compile_source(src)
    rep = autoopt.expand_library(g, registry=X.b200_registry(autoopt.cpu_registry()))
    assert all(k.endswith("_b200") for k in rep.applications)
    assert not [d for d in g.validate() if d.severity == "error"]
    rng = np.random.default_rng(1)
    ev = frontend.oracle._Evaluator(prog, syms)
    ins = {}
    for p in prog.entry.params:
        if p.shape:
            ins[p.name] = rng.uniform(-1, 1, tuple(ev.eval_index(d, frontend.oracle._Frame())
                                                  for d in p.shape))
        elif p.dtype == "f64":
            ins[p.name] = float(rng.uniform(0.5, 1.5))
    ref = frontend.evaluate_program(prog, syms, {k: np.array(v) for k, v in ins.items()})
    ctx = ExecContext(bindings=syms)
    ctx.bind_inputs({k: np.array(v) for k, v in ins.items()})
    out = interpret(g, ctx)
    for k in ref:
        assert np.array_equal(out[k], ref[k]), k
    g2, _ = frontend.compile_source(src)
    rep2 = autoopt.expand_library(g2, registry=X.b200_registry(autoopt.cpu_registry()),
                                  pinned={"matmul": "native", "reduce": "native"})
    assert not any(k.endswith("_b200") for k in rep2.applications)
    _ = sk


def test_install_order_and_patch():
    _sdfgkit()
    from sdfgkit import autoopt
    from sdfgkit.ir import LibKind

    from paper_2107_00555_b200 import expansions as X

    reg = autoopt.cpu_registry()
    X.install(reg)
    assert [x.name for x in reg.by_kind[LibKind.MATMUL]] == ["b200", "blocked_native", "native"]
    assert [x.name for x in reg.by_kind[LibKind.REDUCE]] == ["b200", "tiled_native", "native"]
    orig = autoopt.cpu_registry
    with X.patched_cpu_registry(autoopt):
        assert [x.name for x in autoopt.cpu_registry().by_kind[LibKind.TRANSPOSE]][0] == "b200"
    assert autoopt.cpu_registry is orig


@pytest.mark.gpu
@pytest.mark.parametrize("name,syms", [("atax", {"M": 300, "N": 257}),
                                       ("gemver", {"N": 301}),
                                       ("k3mm", {"NI": 70, "NJ": 65, "NK": 64, "NM": 33, "NL": 90})])
def test_auto_optimize_to_device_through_registry(name, syms):
    """auto_optimize (its pipeline, the b200 registry patched in) -> this
    backend's interpret on the live reference Sdfg object: equal to the
    reference oracle within 1e-12, and the products run as device library
    kernels (row-pass / DMMA), not as expanded WCR maps."""
    _sdfgkit()
    from sdfgkit import autoopt, frontend

    from conftest import rel_err
    from paper_2107_00555_b200 import ExecContext, expansions as X, interpret, machine, plan as P

    src = _corpus(name)
    prog = frontend.parse(src)
    g, _ = frontend.compile_source(src)
    with X.patched_cpu_registry(autoopt):
        autoopt.auto_optimize(g)
    rng = np.random.default_rng(2)
    ev = frontend.oracle._Evaluator(prog, syms)
    ins = {}
    for p in prog.entry.params:
        if p.shape:
            ins[p.name] = rng.uniform(-1, 1, tuple(ev.eval_index(d, frontend.oracle._Frame())
                                                  for d in p.shape))
        elif p.dtype == "f64":
            ins[p.name] = float(rng.uniform(0.5, 1.5))
    ref = frontend.evaluate_program(prog, syms, {k: np.array(v) for k, v in ins.items()})
    out = interpret(g, ExecContext(bindings=syms).bind_inputs(ins))
    for k in ref:
        assert rel_err(out[k], ref[k]) <= 1e-12, k
    ex = next(e for e in machine._exec_cache.values() if e.g.name == g.name)
    libs = [op for op in ex.planner.all_ops if isinstance(op, P.LibOp) and op.kind == "matmul"]
    assert libs
