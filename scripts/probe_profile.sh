#!/bin/bash
# dev tool: full ncu capture of the generic map kernel on heat_3d and jacobi_2d
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python scripts/probe_time.py heat_3d.raw '{"N": 400, "TSTEPS": 3}' 2 > gpurun_out/plain_heat.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:b2_map -s 2 -c 1 -o gpurun_out/prof_heat python scripts/probe_time.py heat_3d.raw '{"N": 400, "TSTEPS": 3}' 2 > gpurun_out/ncu_heat.log 2>&1
python scripts/probe_time.py jacobi_2d.raw '{"N": 2000, "TSTEPS": 3}' 2 > gpurun_out/plain_jac.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:b2_map -s 2 -c 1 -o gpurun_out/prof_jac python scripts/probe_time.py jacobi_2d.raw '{"N": 2000, "TSTEPS": 3}' 2 > gpurun_out/ncu_jac.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
