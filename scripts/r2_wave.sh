#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_config.py -m gpu -x -q -k "heat" 2>&1 | tail -1
for cfg in "0 2 3" "2 3 3" "3 3 3" "6 3 3"; do
  set -- $cfg
  B2_WAVE_TB=$1 B2_WAVE_LAG=$2 B2_WAVE_CTAS=$3 timeout 300 python scripts/bench_suite.py --only heat_3d --reps 10 --out gpurun_out/tune.json 2>&1 | sed "s/^/tb=$1 lag=$2 ctas=$3 /"
done
