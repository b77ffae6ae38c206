python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -o faulthandler_timeout=200 2>&1 | tail -2
for v in raw auto pipe; do timeout -s KILL 300 python scripts/probe_time.py conv2d_bias.$v '{"NB": 8, "H": 256, "W": 256, "CI": 3, "CO": 16, "K": 20, "HO": 237, "WO": 237}' 3 2>&1 | grep -E "rep 2|Error" | head -2; done
