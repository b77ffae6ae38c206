python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python bench.py --workload jacobi_2d_local 2>&1 | grep metric | cut -c1-1200
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -o faulthandler_timeout=200 2>&1 | tail -2
