python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 120 python scripts/probe_time.py jacobi_2d.raw '{"N":2000,"TSTEPS":100}' 3 2>&1 | grep -E 'rep 2|Error' | head -1
timeout -s KILL 120 python scripts/probe_time.py go_fast.pipe '{"N":12000}' 3 2>&1 | grep -E 'rep 2|Error' | head -1
timeout -s KILL 900 python -m pytest tests -m gpu -q -o faulthandler_timeout=200 2>&1 | tail -2
