python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/suite
rm -f profiles/bench_suite_r01_v4.json
timeout -s KILL 1200 python scripts/bench_suite.py --out profiles/bench_suite_r01_v4.json > gpurun_out/suite.log 2>&1; tail -12 gpurun_out/suite.log
cp profiles/bench_suite_r01_v4.json gpurun_out/suite/
timeout -s KILL 300 python bench.py --workload matmul_f32 --steps 3 --warmup 3 2>&1 | grep metric > gpurun_out/suite/summa_f32.json; cut -c1-1500 gpurun_out/suite/summa_f32.json
timeout -s KILL 600 python bench.py --workload matmul --steps 3 --warmup 3 2>&1 | grep metric > gpurun_out/suite/summa_f64.json; cut -c1-300 gpurun_out/suite/summa_f64.json
