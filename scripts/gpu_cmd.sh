python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
python -c "
import sys; sys.path.insert(0,'tests')
from paper_2107_00555_b200 import sdfg
from paper_2107_00555_b200.machine import GpuExecutor
from conftest import GOLDEN
for n,s in (('softmax.raw',{'N':2,'H':3,'SM':64}),('atax.raw',{'M':300,'N':200}),('gemver.raw',{'N':256}),('go_fast.pipe',{'N':300}),('heat_3d.raw',{'N':20,'TSTEPS':2})):
    ex=GpuExecutor(sdfg.load(GOLDEN/'graphs'/(n+'.json')), s); print(n, sorted(ex.zero_skip)); ex.close()
"
for z in 0 1; do echo "== ZERO_SKIP=$z"; B2_ZERO_SKIP=$z timeout -s KILL 300 python scripts/bench_suite.py --only softmax,gemver,atax --reps 10 --out gpurun_out/pf.json 2>&1 | grep -E "ms "; done
timeout -s KILL 900 python -m pytest tests -q -m gpu -rf 2>&1 | grep -E "FAILED|passed|failed|Error" | head -8
timeout -s KILL 300 python scripts/parity_sweep.py 2>&1 | tail -9
