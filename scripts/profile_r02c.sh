#!/bin/bash
# Full ncu captures of the kernels changed last: the softmax row reduction
# with its fused epilogue, the jacobi_2d row march (march2).  Each follows the
# identical plain command exiting 0.
P="python scripts/probe_time.py"
S='{"N": 64, "H": 16, "SM": 512}'
$P softmax.raw "$S" 2 > gpurun_out/p_sm.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:b2_map_softmax_2 -c 1 \
  -o gpurun_out/prof_softmax_r02c $P softmax.raw "$S" 2 > gpurun_out/ncu_sm.log 2>&1
echo "sm rc=$?"
J='{"N": 2000, "TSTEPS": 100}'
$P jacobi_2d.raw "$J" 2 > gpurun_out/p_j.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:b2_map_jacobi_2d_0 -s 5 -c 1 \
  -o gpurun_out/prof_jacobi_r02c $P jacobi_2d.raw "$J" 2 > gpurun_out/ncu_j.log 2>&1
echo "j rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_softmax_r02c.ncu-rep gpurun_out/prof_jacobi_r02c.ncu-rep > gpurun_out/r02c_ncu_summary.json 2>&1
head -60 gpurun_out/r02c_ncu_summary.json
