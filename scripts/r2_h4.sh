#!/bin/bash
# after turning the row-reduction next-row prefetch on: smoke, full GPU suite,
# suite pass, softmax row-kernel ncu capture (after its plain run exits 0)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke.log 2>&1
echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/i_gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/i_gpu_tests.log
timeout 1800 python scripts/bench_suite.py --reps 10 --out gpurun_out/bench_suite_r02i.json > gpurun_out/i_suite.log 2>&1
echo "suite rc=$?"; tail -12 gpurun_out/i_suite.log
P="python scripts/probe_time.py"
S='{"N": 64, "H": 16, "SM": 512}'
$P softmax.raw "$S" 2 > gpurun_out/i_p_sm.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:b2_map_softmax_2 -c 1 \
  -o gpurun_out/prof_softmax_r02i $P softmax.raw "$S" 2 > gpurun_out/i_ncu_sm.log 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_softmax_r02i.ncu-rep > gpurun_out/r02i_ncu_softmax.json 2>&1
head -24 gpurun_out/r02i_ncu_softmax.json
