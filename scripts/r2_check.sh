#!/bin/bash
# round-2 GPU check: contract + config parity tests, BLAS-2 timing with and
# without compensated sums
set -x
python -m pytest tests/test_gpu_contract.py tests/test_gpu_parity.py tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/r2b_tests.log 2>&1
python -m pytest tests/test_gpu_config.py -m gpu -q -s > gpurun_out/r2b_config.log 2>&1
python scripts/bench_suite.py --only atax,bicg,gemver --reps 20 --out gpurun_out/r2b_suite_comp.json > gpurun_out/r2b_suite.log 2>&1
B2_RP_COMP=0 python scripts/bench_suite.py --only atax,bicg,gemver --reps 20 --out gpurun_out/r2b_suite_plain.json >> gpurun_out/r2b_suite.log 2>&1
tail -5 gpurun_out/r2b_tests.log; grep -E "passed|failed|^[a-z_0-9]+ \{" gpurun_out/r2b_config.log | tail -20; cat gpurun_out/r2b_suite.log
