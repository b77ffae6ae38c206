"""Generate the golden fixtures by running the REFERENCE itself.

Run here (the container that has /root/reference), never on the GPU box:

    python tests/golden/make_golden.py

For every kernel — the reference corpus (pkg/tests/corpus/*.dpy, read from
/root/reference at generation time, not copied) and this repo's own DSL
programs in programs/*.dpy (heat_3d and the NPBench-sweep kernels, SURVEY.md
Appendix B) — it writes:

* tests/golden/graphs/<kernel>.<variant>.json — schema-v1 graphs produced by
  the reference (serialize.to_dict, pkg/src/sdfgkit/serialize.py:145):
  ``raw``  = frontend.compile_source (frontend/__init__.py:25-45),
  ``pipe`` = coarsen -> cleanup_maps -> subgraph_fusion (reverted when it
             breaks scope structure) -> transient_mitigation,
  ``auto`` = autoopt.auto_optimize (autoopt.py:990), where it succeeds,
  ``b2reg`` = auto_optimize with this repo's b200 library expansions ahead
             of the CPU ones in the registry (expansions.py).
* tests/golden/vectors/<kernel>.v<i>.s<seed>.npz — inputs drawn with the
  reference conftest's make_inputs semantics (pkg/tests/conftest.py:38-49),
  outputs of the reference oracle ``evaluate_program`` (frontend/oracle.py:37)
  and of the reference interpreter ``interpret`` on the raw graph
  (interp.py:139), plus the interpreter's counters.
* tests/golden/manifest.json — symbols, variants, counters, parameter order.
"""

from __future__ import annotations

import copy
import json
import os
import pathlib
import sys
import traceback

import numpy as np

REF = pathlib.Path(os.environ.get("REF_PKG", "/root/reference/pkg"))
HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF / "src"))

from sdfgkit import autoopt, frontend, passes  # noqa: E402
from sdfgkit.frontend import oracle as ref_oracle  # noqa: E402
from sdfgkit.interp import ExecContext, interpret  # noqa: E402
from sdfgkit.serialize import to_dict  # noqa: E402

# Size variants: the reference oracle suite's desk sizes
# (pkg/tests/test_oracle_suite.py:15-31) plus one odd-sized variant per
# kernel that exercises partial CUDA tiles.
SIZES = {
    "gemm": [{"NI": 4, "NJ": 6, "NK": 8}, {"NI": 8, "NJ": 4, "NK": 6}, {"NI": 37, "NJ": 45, "NK": 29}],
    "jacobi_1d": [{"N": 8, "TSTEPS": 4}, {"N": 6, "TSTEPS": 2}, {"N": 301, "TSTEPS": 5}],
    "jacobi_2d": [{"N": 6, "TSTEPS": 4}, {"N": 8, "TSTEPS": 2}, {"N": 67, "TSTEPS": 4}],
    "atax": [{"M": 6, "N": 4}, {"M": 4, "N": 8}, {"M": 53, "N": 71}],
    "bicg": [{"N": 6, "M": 4}, {"N": 61, "M": 47}],
    "mvt": [{"N": 6}, {"N": 8}, {"N": 57}],
    "gesummv": [{"N": 4}, {"N": 8}, {"N": 49}],
    "gemver": [{"N": 6}, {"N": 41}],
    "k2mm": [{"NI": 4, "NJ": 6, "NK": 8, "NL": 4}, {"NI": 19, "NJ": 23, "NK": 17, "NL": 21}],
    "k3mm": [{"NI": 4, "NJ": 6, "NK": 8, "NM": 4, "NL": 6}],
    "doitgen": [{"NR": 4, "NQ": 4, "NP": 8}, {"NR": 6, "NQ": 4, "NP": 6}],
    "adi": [{"N": 8, "TSTEPS": 2}, {"N": 6, "TSTEPS": 4}],
    "fig4_loop": [{"NI": 4}, {"NI": 8}],
    "wcr_sum": [{"NI": 4, "NJ": 6}, {"NI": 33, "NJ": 70}],
    # repo programs
    "heat_3d": [{"N": 6, "TSTEPS": 3}, {"N": 13, "TSTEPS": 4}],
    "go_fast": [{"N": 8}, {"N": 37}],
    "softmax": [{"N": 2, "H": 2, "SM": 4}, {"N": 1, "H": 3, "SM": 6}],
    "azimint_naive": [{"N": 64, "NPT": 4}, {"N": 301, "NPT": 7}],
    "conv2d_bias": [{"NB": 2, "H": 6, "W": 6, "CI": 2, "CO": 3, "K": 3, "HO": 4, "WO": 4},
                    {"NB": 1, "H": 9, "W": 8, "CI": 3, "CO": 5, "K": 2, "HO": 8, "WO": 7}],
    "nbody": [{"N": 5, "NT": 2}, {"N": 9, "NT": 1}],
    "matmul": [{"M": 4, "K": 6, "N": 5}, {"M": 67, "K": 45, "N": 129}],
    # WCR mul / add-of-negated, sum(A, axis), negative floor division,
    # NaN-ordered min / max (interp.py + texpr.py semantics)
    "wcr_ops": [{"N": 7, "M": 5}, {"N": 33, "M": 70}],
    # REDUCE mul / min / max / full, REDUCE into a WCR-add output, TRANSPOSE
    # (library-node semantics of interp.py:462-480; see mutate_libops)
    "libops": [{"N": 4, "M": 6}, {"N": 37, "M": 53}],
}
ONLY = sys.argv[1:]
CORPUS = ["adi", "atax", "bicg", "doitgen", "fig4_loop", "gemm", "gemver", "gesummv",
          "jacobi_1d", "jacobi_2d", "k2mm", "k3mm", "mvt", "wcr_sum"]
REPO_PROGRAMS = ["heat_3d", "go_fast", "softmax", "azimint_naive", "conv2d_bias", "nbody",
                 "matmul", "wcr_ops", "libops"]


def mutate_libops(g):
    """The DSL only lowers ``sum`` (REDUCE add, lower.py:268-282) and has no
    transpose, so the library-node variants the interpreter supports are
    made here on the compiled graph: REDUCE op mul (s0) / min (s1) / max
    (s2, s4 full), a WCR-add output (s3: u += row sums), and a TRANSPOSE
    state B = A.T appended after s4.  Their expected values come from the
    reference interpreter (interp.py:462-480), the oracle has no such ops."""
    from sdfgkit.ir import AccessNode, InterstateEdge, LibKind, LibraryNode, Memlet, Wcr
    from sdfgkit.symbolic import SubsetRange, Sym

    ops = {"s0": "mul", "s1": "min", "s2": "max", "s4": "max"}
    for st in g.states:
        for n in st.nodes.values():
            if isinstance(n, LibraryNode) and n.kind is LibKind.REDUCE:
                if st.label in ops:
                    n.attributes["op"] = ops[st.label]
                if st.label == "s3":
                    for e in st.out_edges(n):
                        e.memlet.wcr = Wcr.ADD
    last = g.states[-1].label
    st = g.add_state("s_transpose")
    a = st.add(AccessNode("A"))
    tr = st.add(LibraryNode(LibKind.TRANSPOSE, "transpose", {}))
    b = st.add(AccessNode("B"))
    st.add_edge(a, tr, Memlet("A", SubsetRange.full((Sym("N"), Sym("M")))), dst_conn="a")
    st.add_edge(tr, b, Memlet("B", SubsetRange.full((Sym("M"), Sym("N")))), src_conn="out")
    g.transitions.append(InterstateEdge(last, "s_transpose"))
    return g


MUTATE = {"libops": mutate_libops}


def b200_registry_variant(g):
    """auto_optimize with the b200 library expansions first in the registry
    (paper_2107_00555_b200/expansions.py): MATMUL / REDUCE / TRANSPOSE stay
    device library nodes (inside single-node wrappers)."""
    sys.path.insert(0, str(REPO))
    from paper_2107_00555_b200 import expansions

    with expansions.patched_cpu_registry(autoopt):
        autoopt.auto_optimize(g)
    return g
SEEDS = (0, 1)


def source(name: str) -> str:
    if name in CORPUS:
        return (REF / "tests" / "corpus" / f"{name}.dpy").read_text()
    return (REPO / "programs" / f"{name}.dpy").read_text()


def eval_shape(expr, symbols):
    ev = ref_oracle._Evaluator(frontend.Program([], ""), symbols)
    return ev.eval_index(expr, ref_oracle._Frame())


def make_inputs(program, symbols, seed):
    # pkg/tests/conftest.py:38-49 semantics
    rng = np.random.default_rng(seed)
    inputs = {}
    for p in program.entry.params:
        if p.shape:
            shape = tuple(eval_shape(d, symbols) for d in p.shape)
            inputs[p.name] = rng.uniform(-1.0, 1.0, size=shape)
        elif p.dtype == "f64":
            inputs[p.name] = float(rng.uniform(0.5, 1.5))
    return inputs


def pipeline(g):
    """SURVEY.md §7 GPU pre-pipeline."""
    passes.coarsen(g)
    autoopt.cleanup_maps(g)
    fused = False
    trial = copy.deepcopy(g)
    try:
        autoopt.subgraph_fusion(trial)
        if not [d for d in trial.validate() if d.severity == "error"]:
            for st in trial.states:
                st.scope_parents()
            g = trial
            fused = True
    except Exception:  # noqa: BLE001 — reference bug
        pass
    autoopt.transient_mitigation(g)
    errs = [d for d in g.validate() if d.severity == "error"]
    assert not errs, errs
    return g, fused


def main():
    gdir = HERE / "graphs"
    vdir = HERE / "vectors"
    gdir.mkdir(exist_ok=True)
    vdir.mkdir(exist_ok=True)
    mpath = HERE / "manifest.json"
    manifest = json.loads(mpath.read_text()) if (ONLY and mpath.exists()) else {"kernels": {}}
    for name in CORPUS + REPO_PROGRAMS:
        if ONLY and name not in ONLY:
            continue
        src = source(name)
        program = frontend.parse(src)
        g, diags = frontend.compile_source(src)
        assert g is not None, [str(d) for d in diags]
        if name in MUTATE:
            g = MUTATE[name](g)
        variants = {"raw": copy.deepcopy(g)}
        gp, fused = pipeline(copy.deepcopy(g))
        variants["pipe"] = gp
        try:
            ga = copy.deepcopy(g)
            autoopt.auto_optimize(ga)
            variants["auto"] = ga
        except Exception as ex:  # noqa: BLE001
            print(f"[{name}] auto_optimize failed: {ex}")
        try:
            variants["b2reg"] = b200_registry_variant(copy.deepcopy(g))
        except Exception as ex:  # noqa: BLE001
            print(f"[{name}] auto_optimize with the b200 registry failed: {ex}")
        for v, gg in variants.items():
            (gdir / f"{name}.{v}.json").write_text(json.dumps(to_dict(gg), indent=1) + "\n")
        entry = {
            "params": [p.name for p in program.entry.params],
            "scalars": [p.name for p in program.entry.params if not p.shape and p.dtype == "f64"],
            "variants": sorted(variants),
            "pipe_fused": fused,
            "cases": [],
        }
        for vi, syms in enumerate(SIZES[name]):
            for seed in SEEDS:
                inputs = make_inputs(program, syms, seed)
                if name in MUTATE:  # library ops the oracle cannot express
                    octx = ExecContext(bindings=dict(syms))
                    octx.bind_inputs({k: np.array(v) if hasattr(v, "shape") else v
                                      for k, v in inputs.items()})
                    ref = interpret(copy.deepcopy(variants["raw"]), octx)
                else:
                    ref = ref_oracle.evaluate_program(
                        program, syms,
                        {k: (np.array(v, copy=True) if hasattr(v, "shape") else v)
                         for k, v in inputs.items()})
                blob = {}
                for k, v in inputs.items():
                    blob[f"in/{k}"] = np.asarray(v, dtype=np.float64)
                for k, v in ref.items():
                    blob[f"oracle/{k}"] = np.asarray(v)
                counters, same = {}, {}
                for vname, gg in variants.items():
                    ctx = ExecContext(bindings=dict(syms))
                    ctx.bind_inputs({k: np.array(v) if hasattr(v, "shape") else v
                                     for k, v in inputs.items()})
                    try:
                        out = interpret(gg, ctx)
                    except Exception:  # noqa: BLE001
                        traceback.print_exc()
                        continue
                    counters[vname] = ctx.counters.as_dict()
                    for k, v in out.items():
                        blob[f"interp_{vname}/{k}"] = np.asarray(v)
                    same[vname] = bool(all(np.array_equal(out[k], ref[k], equal_nan=True) for k in ref))
                fname = f"{name}.v{vi}.s{seed}.npz"
                np.savez_compressed(vdir / fname, **blob)
                entry["cases"].append({"file": fname, "symbols": syms, "seed": seed,
                                       "counters": counters, "interp_equals_oracle": same})
                print(f"[{name}] v{vi} seed{seed}: interp==oracle {same}")
        manifest["kernels"][name] = entry
    (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")


if __name__ == "__main__":
    main()
