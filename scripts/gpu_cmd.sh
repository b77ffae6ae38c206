python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 120 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" -o faulthandler_timeout=60 2>&1 | tail -2
for g in 1 8 16; do echo "group $g"; B2_DGEMM_GROUP=$g timeout -s KILL 200 python bench.py --workload matmul --steps 3 --warmup 3 2>&1 | grep metric | cut -c1-150; done
