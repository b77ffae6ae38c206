python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -q -m gpu -rf 2>&1 | grep -E "FAILED|passed|failed|Error" | head -8
timeout -s KILL 300 python scripts/bench_suite.py --only gemver,atax,bicg,go_fast,jacobi_2d,nbody --reps 10 --out gpurun_out/pf.json 2>&1 | grep -E "ms "
