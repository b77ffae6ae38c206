timeout 300 python scripts/probe_dgemm.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dgemm -s 4 -c 1 -o gpurun_out/dgemm_final python scripts/probe_dgemm.py > gpurun_out/ncu_dgf.log 2>&1
tail -2 gpurun_out/ncu_dgf.log
