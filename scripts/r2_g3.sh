for m in 4 2 3 6; do B2_ROWRED_EPI_MINB=$m timeout 300 python scripts/bench_suite.py --only softmax --reps 10 --out gpurun_out/sm.json 2>&1 | grep softmax | sed "s/^/minb=$m /"; done
