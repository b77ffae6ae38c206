python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q -o faulthandler_timeout=200 2>&1 | tail -2
timeout -s KILL 200 python scripts/probe_time.py nbody.raw '{"N":100,"NT":1000}' 3 2>&1 | grep -E "rep 2|Error" | head -2
timeout -s KILL 200 python scripts/probe_time.py go_fast.pipe '{"N":12000}' 3 2>&1 | grep -E "rep 2|Error" | head -2
timeout -s KILL 200 python scripts/probe_time.py azimint_naive.raw '{"N": 1000000, "NPT": 1000}' 3 2>&1 | grep -E "rep 2|Error" | head -2
