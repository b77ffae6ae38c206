python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python scripts/parity_sweep.py > gpurun_out/parity_sweep.log 2>&1; echo rc=$?
tail -30 gpurun_out/parity_sweep.log
