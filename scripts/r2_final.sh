#!/bin/bash
# Round-2 closing batch on one B200: smoke, driver-style bench lines (ours +
# reference arm), bench suite, launch list of the bench command (the ncu pass
# runs only after the identical plain command exited 0).
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.log 2>&1
echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_ref.log 2>&1
echo "ref rc=$?"
timeout 1800 python scripts/bench_suite.py --reps 10 --out gpurun_out/bench_suite_r02g.json > gpurun_out/f_suite.log 2>&1
echo "suite rc=$?"
S="python bench.py --steps 2 --warmup 3"
timeout 600 $S > gpurun_out/f_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/f_launches.csv $S > gpurun_out/f_ncu.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/f_smoke.log
grep '^{' gpurun_out/f_bench.log gpurun_out/f_bench_ref.log | cut -c1-1200
cat gpurun_out/f_suite.log | tail -12
# the multi-GPU code path (slab runner, NCCL communicator of one rank) on this one GPU
B2_FORCE_SLAB=1 timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/f_slab1.log 2>&1
echo "slab1 rc=$?"
grep '^{' gpurun_out/f_slab1.log | cut -c1-600
