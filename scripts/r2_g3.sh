timeout 600 python scripts/bench_suite.py --only azimint_naive,nbody --reps 5 --out gpurun_out/s_az.json 2>&1 | grep -E "azimint|nbody"
B2_RED_OUT_BLOCK=8 timeout 600 python scripts/bench_suite.py --only azimint_naive --reps 5 --out gpurun_out/s_az8.json 2>&1 | grep -E "azimint"
B2_RED_OUT_BLOCK=1 timeout 600 python scripts/bench_suite.py --only azimint_naive --reps 5 --out gpurun_out/s_az1.json 2>&1 | grep -E "azimint"
timeout 1500 python -m pytest tests -m gpu -q -x -k "azimint or reduce or wcr or nbody or config or parity" 2>&1 | tail -2
