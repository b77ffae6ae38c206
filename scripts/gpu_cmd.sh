python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/suite
rm -f profiles/bench_suite_r01_v5.json
timeout -s KILL 1200 python scripts/bench_suite.py --out profiles/bench_suite_r01_v5.json > gpurun_out/suite.log 2>&1; tail -12 gpurun_out/suite.log
cp profiles/bench_suite_r01_v5.json gpurun_out/suite/
