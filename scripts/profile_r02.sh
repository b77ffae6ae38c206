#!/bin/bash
python scripts/bench_suite.py --reps 10 --out gpurun_out/bench_suite_r02.json > gpurun_out/bench_suite_r02.log 2>&1
cat gpurun_out/bench_suite_r02.log
