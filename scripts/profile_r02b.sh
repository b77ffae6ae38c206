#!/bin/bash
# Round-2 (b) full ncu captures of the kernels changed late in the round:
# the 256-row DMMA contraction (conv2d_bias), the 32-deep DGEMM (4096^3), the
# persistent TF32 pair GEMM at a SUMMA 4x2 panel shape.  Each capture follows
# the identical plain command exiting 0.
C='{"NB": 8, "H": 256, "W": 256, "CI": 3, "CO": 16, "K": 20, "HO": 237, "WO": 237}'
P="python scripts/probe_time.py"
$P conv2d_bias.raw "$C" 2 > gpurun_out/p_conv.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2_map_conv2d_bias_1 -s 1 -c 1 \
  -o gpurun_out/prof_conv2d_r02b $P conv2d_bias.raw "$C" 2 > gpurun_out/ncu_conv.log 2>&1
echo "conv rc=$?"
timeout 300 python scripts/probe_dgemm.py > gpurun_out/p_dgemm.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_dmma -c 1 \
  -o gpurun_out/prof_dgemm_r02b python scripts/probe_dgemm.py > gpurun_out/ncu_dgemm.log 2>&1
echo "dgemm rc=$?"
timeout 300 python scripts/probe_tcgemm.py > gpurun_out/p_tc.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_sgemm_pair -s 18 -c 1 \
  -o gpurun_out/prof_tcpair_r02b python scripts/probe_tcgemm.py > gpurun_out/ncu_tc.log 2>&1
echo "tc rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_conv2d_r02b.ncu-rep gpurun_out/prof_dgemm_r02b.ncu-rep gpurun_out/prof_tcpair_r02b.ncu-rep > gpurun_out/r02b_ncu_summary.json 2>&1
cat gpurun_out/r02b_ncu_summary.json | head -80
