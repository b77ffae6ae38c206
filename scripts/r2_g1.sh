timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/g1_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/g1_tests.log
./scripts/heatlab/heatlab 40 > gpurun_out/g1_heatlab.log 2>&1; echo "lab rc=$?"
cat gpurun_out/g1_heatlab.log
