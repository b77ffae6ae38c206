for m in 2 4; do B2_ROWRED_EPI_MINB=$m timeout 300 python scripts/bench_suite.py --only softmax --reps 10 --out gpurun_out/sm.json 2>&1 | grep softmax | sed "s/^/prologue minb=$m /"; done
