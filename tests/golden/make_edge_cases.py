"""Edge-case fixtures made by running the REFERENCE itself (here, never on the
GPU box): degenerate sizes the desk-size goldens do not reach — empty
interiors (N = 2 stencils), loops that never iterate (TSTEPS = 1),
single-element and rank-1 matrices, one-row / one-column operands, one
particle, one bin.

    python tests/golden/make_edge_cases.py

For every case it runs the reference interpreter (interp.py:139) on the raw
graph already committed under tests/golden/graphs/ and, where the DSL can
express it, the reference oracle evaluate_program (frontend/oracle.py:37),
and writes tests/golden/edges/<kernel>.e<i>.npz (in/…, interp/…, oracle/…)
plus tests/golden/edges/manifest.json.  A case the reference itself rejects
is recorded with its error message (the B200 executor must then raise too).
"""

from __future__ import annotations

import importlib
import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
argv, sys.argv = sys.argv, sys.argv[:1]
MG = importlib.import_module("make_golden")  # reference imports + input semantics
sys.argv = argv

from sdfgkit import frontend  # noqa: E402
from sdfgkit.frontend import oracle as ref_oracle  # noqa: E402
from sdfgkit.interp import ExecContext, interpret  # noqa: E402

ser = importlib.import_module("sdfgkit.serialize")

CASES = {
    "jacobi_2d": [{"N": 2, "TSTEPS": 3}, {"N": 3, "TSTEPS": 1}, {"N": 3, "TSTEPS": 2}],
    "jacobi_1d": [{"N": 2, "TSTEPS": 3}, {"N": 3, "TSTEPS": 2}],
    "heat_3d": [{"N": 2, "TSTEPS": 2}, {"N": 3, "TSTEPS": 1}, {"N": 3, "TSTEPS": 3}],
    "gemm": [{"NI": 1, "NJ": 1, "NK": 1}, {"NI": 1, "NJ": 5, "NK": 1}, {"NI": 3, "NJ": 1, "NK": 7}],
    "atax": [{"M": 1, "N": 1}, {"M": 1, "N": 9}, {"M": 9, "N": 1}],
    "bicg": [{"N": 1, "M": 1}, {"N": 7, "M": 1}],
    "mvt": [{"N": 1}],
    "gesummv": [{"N": 1}],
    "gemver": [{"N": 1}, {"N": 2}],
    "k2mm": [{"NI": 1, "NJ": 1, "NK": 1, "NL": 1}],
    "doitgen": [{"NR": 1, "NQ": 1, "NP": 1}, {"NR": 1, "NQ": 3, "NP": 2}],
    "fig4_loop": [{"NI": 1}],
    "wcr_sum": [{"NI": 1, "NJ": 1}, {"NI": 1, "NJ": 17}],
    "softmax": [{"N": 1, "H": 1, "SM": 1}],
    "go_fast": [{"N": 1}],
    "azimint_naive": [{"N": 5, "NPT": 1}],
    "nbody": [{"N": 1, "NT": 1}, {"N": 2, "NT": 1}],
    "matmul": [{"M": 1, "K": 1, "N": 1}, {"M": 1, "K": 33, "N": 1}],
    "conv2d_bias": [{"NB": 1, "H": 2, "W": 2, "CI": 1, "CO": 1, "K": 1, "HO": 2, "WO": 2}],
    "wcr_ops": [{"N": 1, "M": 1}],
    "libops": [{"N": 1, "M": 1}],
}
SEED = 11


def main():
    out = HERE / "edges"
    out.mkdir(exist_ok=True)
    manifest = {}
    for name, cases in CASES.items():
        src = MG.source(name)
        program = frontend.parse(src)
        doc = json.loads((HERE / "graphs" / f"{name}.raw.json").read_text())
        entry = []
        for i, syms in enumerate(cases):
            inputs = MG.make_inputs(program, syms, SEED)
            blob = {f"in/{k}": np.asarray(v, dtype=np.float64) for k, v in inputs.items()}
            rec = {"file": f"{name}.e{i}.npz", "symbols": syms}
            try:
                ctx = ExecContext(bindings=dict(syms))
                ctx.bind_inputs({k: np.array(v) if hasattr(v, "shape") else v
                                 for k, v in inputs.items()})
                res = interpret(ser.from_dict(doc), ctx)
                for k, v in res.items():
                    blob[f"interp/{k}"] = np.asarray(v)
                rec["counters"] = ctx.counters.as_dict()
            except Exception as ex:  # noqa: BLE001 - the reference rejects it
                rec["reference_error"] = f"{type(ex).__name__}: {ex}"
            if name not in MG.MUTATE and "reference_error" not in rec:
                try:
                    ref = ref_oracle.evaluate_program(
                        program, syms, {k: (np.array(v, copy=True) if hasattr(v, "shape") else v)
                                        for k, v in inputs.items()})
                    for k, v in ref.items():
                        blob[f"oracle/{k}"] = np.asarray(v)
                except Exception as ex:  # noqa: BLE001
                    rec["oracle_error"] = f"{type(ex).__name__}: {ex}"
            np.savez_compressed(out / rec["file"], **blob)
            entry.append(rec)
            print(name, syms, rec.get("reference_error", "ok"), rec.get("oracle_error", ""))
        manifest[name] = entry
    (out / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")


if __name__ == "__main__":
    main()
