python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
run() { echo "== $*"; env "$@" timeout -s KILL 300 python scripts/bench_suite.py --only heat_3d --reps 10 --out gpurun_out/pf.json 2>&1 | grep -E "ms " | tail -1; }
for i in 1 2 3; do run B2_SWEEP_ALTERNATE=0; run B2_SWEEP_ALTERNATE=1; done
timeout -s KILL 600 python -m pytest tests -q -m gpu -rf -k "heat" 2>&1 | tail -2
