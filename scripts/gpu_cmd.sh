python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
B2_RP_COOP=1 timeout -s KILL 120 python scripts/probe_time.py atax.raw '{"M": 8000, "N": 8000}' 3 2>&1 | tail -4
run() { echo "== $*"; env "$@" timeout -s KILL 200 python scripts/bench_suite.py --only gemver,atax,bicg --reps 10 --out gpurun_out/pf.json 2>&1 | grep -E "ms "; }
for i in 1 2; do run B2_RP_COOP=0; run B2_RP_COOP=1; done
B2_RP_COOP=1 timeout -s KILL 600 python -m pytest tests -q -m gpu -rf -k "blas2 or atax or bicg or gemver or gesummv or mvt or parity" 2>&1 | grep -E "FAILED|passed|failed|Error" | head -8
B2_RP_COOP=1 timeout -s KILL 300 python scripts/parity_sweep.py 2>&1 | grep -E "atax|bicg|gemver|FAILS"
