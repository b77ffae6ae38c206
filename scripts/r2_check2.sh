#!/bin/bash
set -x
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r2c_tests.log 2>&1
python -m pytest tests/test_gpu_config.py -m gpu -q -s > gpurun_out/r2c_config.log 2>&1
B2_RP_COMP=0 python -m pytest tests/test_gpu_config.py -m gpu -q -s -k "atax or bicg" > gpurun_out/r2c_config_plain.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r2c_bench_tma3.log 2>&1
B2_TMA3=0 python bench.py --steps 10 --warmup 3 > gpurun_out/r2c_bench_march.log 2>&1
python scripts/peaks/measure_peaks.py gpurun_out/r2c_peaks.json > gpurun_out/r2c_peaks.log 2>&1
tail -3 gpurun_out/r2c_tests.log; grep -E "passed|failed|^[a-z_0-9]+ \{" gpurun_out/r2c_config.log gpurun_out/r2c_config_plain.log
python - <<'PY'
import json
for f in ("gpurun_out/r2c_bench_tma3.log", "gpurun_out/r2c_bench_march.log"):
    for ln in open(f):
        if ln.startswith("{"):
            d = json.loads(ln); print(f, d["value"], d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["launch_ms"], d["roofline"]["frac"], d["clocks"])
PY
cat gpurun_out/r2c_peaks.json
