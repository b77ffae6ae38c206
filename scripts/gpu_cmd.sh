python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -o faulthandler_timeout=200 2>&1 | tail -2
for p in 0 1; do echo "PDL=$p"
B2_PDL=$p timeout -s KILL 120 python scripts/probe_time.py jacobi_2d.raw '{"N":2000,"TSTEPS":100}' 3 2>&1 | grep -E "rep 2|Error" | head -1
B2_PDL=$p timeout -s KILL 120 python scripts/probe_time.py nbody.raw '{"N":100,"NT":1000}' 3 2>&1 | grep -E "rep 2|Error" | head -1
B2_PDL=$p timeout -s KILL 120 python scripts/probe_time.py heat_3d.raw '{"N":400,"TSTEPS":100}' 3 2>&1 | grep -E "rep 2|Error" | head -1
B2_PDL=$p timeout -s KILL 120 python scripts/probe_time.py gemver.raw '{"N":8000}' 3 2>&1 | grep -E "rep 2|Error" | head -1
done
