#!/bin/bash
python -m pytest tests/test_gpu_config.py tests/test_gpu_contract.py -m gpu -q -s > gpurun_out/r2d_config.log 2>&1
B2_RP_COMP=1 python -m pytest tests/test_gpu_config.py -m gpu -q -s -k "atax or bicg" > gpurun_out/r2d_config_comp.log 2>&1
grep -E "passed|failed|^[a-z_0-9 -]+ \{|Error" gpurun_out/r2d_config.log gpurun_out/r2d_config_comp.log | cut -c1-400
