timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config.py tests/test_gpu_kernels.py tests/test_gpu_contract.py -m gpu -q -x -k "gemver or atax or bicg or mvt or gesummv or rowpass or blas" 2>&1 | tail -1
for r in 0 1 0 1; do B2_RP_REV=$r timeout 300 python scripts/bench_suite.py --only gemver --reps 20 --out gpurun_out/gv.json 2>&1 | grep gemver | sed "s/^/rev=$r /"; done
