python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
run() { echo "== $*"; env "$@" timeout -s KILL 600 python scripts/bench_suite.py --only softmax,heat_3d,go_fast,nbody,conv2d_bias,jacobi_2d --out gpurun_out/sm.json 2>&1 | grep -E "ms "; python -c "
import json; d=json.load(open('gpurun_out/sm.json'))['softmax']['kernels']; print({k:round(v['ms_total'],3) for k,v in d.items()})"; }
run B2_FORWARD=1
run B2_FORWARD=0
timeout -s KILL 900 python -m pytest tests -q -m gpu -rf -o faulthandler_timeout=300 2>&1 | grep -E "FAILED|passed|failed|Error" | head -8
