#!/bin/bash
# pref cw tj chunk
for cfg in "2 8 8 32" "2 8 16 24" "2 8 16 48" "3 8 16 32" "2 4 8 32" "2 4 16 32" "2 16 16 32" "2 8 8 24"; do
  set -- $cfg
  B2_TMA3_PREF=$1 B2_TMA3_CW=$2 B2_TMA3_TJ=$3 B2_TMA3_CHUNK=$4 timeout 300 python scripts/bench_suite.py --only heat_3d --reps 10 --out gpurun_out/tune.json 2>&1 | sed "s/^/pref=$1 cw=$2 tj=$3 chunk=$4 /"
done
