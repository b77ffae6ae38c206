"""Two heat_3d sweeps at N=400 through interpret() (profiling driver)."""
import sys
import pathlib
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2107_00555_b200 import ExecContext, interpret, sdfg  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 400
g = sdfg.load(ROOT / "tests" / "golden" / "graphs" / "heat_3d.raw.json")
rng = np.random.default_rng(0)
ins = {"A": rng.uniform(-1, 1, (N, N, N)), "B": rng.uniform(-1, 1, (N, N, N))}
for _ in range(2):
    interpret(g, ExecContext(bindings={"N": N, "TSTEPS": 2}).bind_inputs(ins))
print("ok")
