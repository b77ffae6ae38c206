#!/bin/bash
# Launch list of the bench command + full ncu captures of the dominant kernels.
# Each ncu run follows the identical plain command exiting 0 (profiling recipe).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 2 --warmup 1"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
P="python scripts/probe_time.py"
$P heat_3d.raw '{"N": 400, "TSTEPS": 3}' 2 > gpurun_out/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:b2_map_heat -s 2 -c 1 -o gpurun_out/prof_heat $P heat_3d.raw '{"N": 400, "TSTEPS": 3}' 2 > gpurun_out/ncu1.log 2>&1
$P bicg.raw '{"N": 8000, "M": 8000}' 2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:b2_rp_bicg -s 1 -c 1 -o gpurun_out/prof_bicg $P bicg.raw '{"N": 8000, "M": 8000}' 2 > gpurun_out/ncu2.log 2>&1
$P gemver.raw '{"N": 8000}' 2 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:b2_rp_gemver_0 -s 1 -c 1 -o gpurun_out/prof_gemver $P gemver.raw '{"N": 8000}' 2 > gpurun_out/ncu3.log 2>&1
$P matmul.raw '{"M": 4096, "K": 4096, "N": 4096}' 2 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dgemm -s 1 -c 1 -o gpurun_out/prof_dgemm $P matmul.raw '{"M": 4096, "K": 4096, "N": 4096}' 2 > gpurun_out/ncu4.log 2>&1
python scripts/probe_sgemm.py 4096 2 > gpurun_out/plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_sgemm -s 1 -c 1 -o gpurun_out/prof_tcsgemm python scripts/probe_sgemm.py 4096 2 > gpurun_out/ncu5.log 2>&1
echo done
