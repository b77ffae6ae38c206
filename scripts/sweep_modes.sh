#!/bin/bash
# dev tool: time the heat_3d / jacobi_2d sweep kernels under each codegen mode
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in $CFGS; do
  set -- $cfg
  echo "== mode $1 vec $2"
  B2_FORCE_MODE=$1 B2_VEC=$2 timeout 120 python scripts/probe_time.py heat_3d.raw '{"N":400,"TSTEPS":20}' 2 2>&1 | grep -E "kernel|Error" | head -2
  [ -n "$JAC" ] && B2_FORCE_MODE=$1 B2_VEC=$2 timeout 120 python scripts/probe_time.py jacobi_2d.raw '{"N":2000,"TSTEPS":20}' 2 2>&1 | grep -E "kernel|Error" | head -2
done
