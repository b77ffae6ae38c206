python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in 0 1 0 1; do echo "STCS=$v"
B2_STCS=$v timeout -s KILL 120 python scripts/probe_time.py heat_3d.raw '{"N":400,"TSTEPS":100}' 3 2>&1 | grep -E "rep 2|Error" | head -1
B2_STCS=$v timeout -s KILL 120 python scripts/probe_time.py go_fast.pipe '{"N":12000}' 3 2>&1 | grep -E "rep 2|Error" | head -1
B2_STCS=$v timeout -s KILL 120 python scripts/probe_time.py softmax.raw '{"N": 64, "H": 16, "SM": 512}' 3 2>&1 | grep -E "rep 2|Error" | head -1
done
