python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout -s KILL 600 python scripts/bench_suite.py --out gpurun_out/bench_suite_r01_v8.json 2>&1 | grep -E "ms "
timeout -s KILL 300 python bench.py > gpurun_out/bench_line_v9.json 2> gpurun_out/bench_err.log; tail -1 gpurun_out/bench_line_v9.json | head -c 300; echo
timeout -s KILL 300 python bench.py --impl reference > gpurun_out/bench_ref_v9.json 2>> gpurun_out/bench_err.log; tail -1 gpurun_out/bench_ref_v9.json | head -c 200; echo
