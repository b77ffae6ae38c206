python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -rf -k "overwritten" 2>&1 | tail -2
