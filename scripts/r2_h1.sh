#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1
echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/h_gpu_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/h_gpu_tests.log
