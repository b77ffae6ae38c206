python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q -o faulthandler_timeout=200 2>&1 | tail -2
