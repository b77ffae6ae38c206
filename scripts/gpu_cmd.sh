python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 600 python scripts/parity_sweep.py 2>&1 | tail -16
