python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 600 python scripts/scaling_projection.py > gpurun_out/scaling_projection.log 2>&1; cat gpurun_out/scaling_projection.log | tail -12
timeout -s KILL 300 python bench.py 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
