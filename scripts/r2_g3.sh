for cfg in "16 4" "16 2" "16 1" "12 2" "20 2" "24 2"; do set -- $cfg
  B2_MARCH2_V=$1 B2_MARCH2_BY=$2 timeout 300 python scripts/bench_suite.py --only jacobi_2d --reps 20 --out gpurun_out/j.json 2>&1 | grep jacobi | sed "s/^/V=$1 BY=$2 /"
done
