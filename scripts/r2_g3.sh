timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for v in "1 0" "1 1" "0 0"; do set -- $v
  B2_MARCH2=$1 B2_MARCH2_PDL=$2 timeout 300 python scripts/bench_suite.py --only jacobi_2d --reps 20 --out gpurun_out/j.json 2>&1 | grep jacobi | sed "s/^/march2=$1 pdl=$2 /"
done
