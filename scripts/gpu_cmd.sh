python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
run() { echo "== $*"; env "$@" timeout -s KILL 300 python scripts/bench_suite.py --only softmax --reps 10 --out gpurun_out/sm.json 2>&1 | grep -E "ms "; python -c "
import json; d=json.load(open('gpurun_out/sm.json'))['softmax']['kernels']; print({k:round(v['ms_total'],3) for k,v in d.items()})"; }
for i in 1 2; do run B2_ROWRED_MINB=8; run B2_ROWRED_MINB=7; done
