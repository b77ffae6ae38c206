#!/bin/bash
# Round-2 closing batch (session h, rebuilt libb2): driver-style bench lines
# (ours + reference arm), bench suite with minimum-traffic softmax bytes,
# launch list of the bench command, one full ncu capture of the headline
# sweep kernel.  Every ncu pass follows the identical plain command exiting 0.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/h_bench.log 2>&1
echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/h_bench_ref.log 2>&1
echo "ref rc=$?"
timeout 1800 python scripts/bench_suite.py --reps 10 --out gpurun_out/bench_suite_r02h.json > gpurun_out/h_suite.log 2>&1
echo "suite rc=$?"
S="python bench.py --steps 2 --warmup 3"
timeout 600 $S > gpurun_out/h_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/h_launches.csv $S > gpurun_out/h_ncu.log 2>&1
echo "launches rc=$?"
P="python scripts/probe_time.py"
H='{"N": 400, "TSTEPS": 100}'
timeout 600 $P heat_3d.raw "$H" 2 > gpurun_out/h_p_heat.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:b2_map_heat_3d_0 -s 5 -c 1 \
  -o gpurun_out/prof_heat_r02h $P heat_3d.raw "$H" 2 > gpurun_out/h_ncu_heat.log 2>&1
echo "ncu heat rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_heat_r02h.ncu-rep > gpurun_out/r02h_ncu_full_summary.json 2>&1
grep '^{' gpurun_out/h_bench.log gpurun_out/h_bench_ref.log | cut -c1-900
tail -14 gpurun_out/h_suite.log
head -30 gpurun_out/r02h_ncu_full_summary.json
