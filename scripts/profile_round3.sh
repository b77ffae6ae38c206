#!/bin/bash
# Pass "f": bench launch list + full captures of the prefetching 64x8 heat
# march kernel and the register-blocked conv2d reduction.  Each ncu run
# follows the identical plain command exiting 0 (profiling recipe).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 2 --warmup 1"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
P="python scripts/probe_time.py"
$P heat_3d.raw '{"N": 400, "TSTEPS": 3}' 2 > gpurun_out/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:b2_map_heat -s 2 -c 1 -o gpurun_out/prof_heat_f $P heat_3d.raw '{"N": 400, "TSTEPS": 3}' 2 > gpurun_out/ncu1.log 2>&1
C='{"NB": 8, "H": 256, "W": 256, "CI": 3, "CO": 16, "K": 20, "HO": 237, "WO": 237}'
$P conv2d_bias.raw "$C" 2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:b2_map_conv2d_bias_1 -s 1 -c 1 -o gpurun_out/prof_conv2d_f $P conv2d_bias.raw "$C" 2 > gpurun_out/ncu2.log 2>&1
echo done
