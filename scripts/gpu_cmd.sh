python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for c in 128 256 0; do echo "chunk $c"; B2_TC_CHUNK=$c timeout -s KILL 60 python scripts/tc_accuracy.py; done
timeout -s KILL 120 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" -o faulthandler_timeout=60 2>&1 | tail -3
for c in 128 256; do B2_TC_CHUNK=$c timeout -s KILL 200 python bench.py --workload matmul_f32 --steps 3 --warmup 3 2>&1 | grep metric | cut -c1-200; done
