"""Write the march kernel the executor generates for heat_3d N=400 (and an
aligned variant when B2_MARCH_ALIGN is set) to gen_heat.cuh for heatlab."""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2107_00555_b200 import codegen as CG, plan as P, sdfg as S  # noqa: E402

syms = {"N": 400, "TSTEPS": 100}
g = S.load(ROOT / "tests" / "golden" / "graphs" / "heat_3d.raw.json")
pl = P.Planner(g, syms).build()
grp = next(o for o in pl.all_ops if isinstance(o, P.MapGroup))
sp = CG.generate(pl, grp, pl.shapes(syms), "gen_heat")
print(sp.block, sp.vec, sp.align, CG.launch_geometry(sp, [398, 398, 398]))
out = pathlib.Path(__file__).with_name("gen_heat.cuh")
out.write_text(sp.source)
