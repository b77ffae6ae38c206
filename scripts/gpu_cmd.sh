python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -q -m gpu -rf -o faulthandler_timeout=300 2>&1 | tail -15
for i in 1 2; do timeout -s KILL 300 python scripts/bench_suite.py --only heat_3d --reps 10 --out gpurun_out/x.json 2>&1 | grep -E "ms "; done
