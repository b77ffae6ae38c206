python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
run() { echo "== $*"; env "$@" timeout -s KILL 300 python scripts/bench_suite.py --only gemver,atax,bicg,azimint_naive,go_fast --reps 10 --out gpurun_out/j.json 2>&1 | grep -E "ms "; }
run B2_RP_PDL=1 B2_FIN_PDL=1
run B2_RP_PDL=0 B2_FIN_PDL=0
run B2_RP_PDL=1 B2_FIN_PDL=1
timeout -s KILL 900 python -m pytest tests -q -m gpu -rf -o faulthandler_timeout=300 2>&1 | grep -E "FAILED|passed|failed|Error" | head -8
