python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout -s KILL 900 python -m pytest tests -q -m gpu -rf 2>&1 | grep -E "FAILED|passed|failed|Error" | head -8
timeout -s KILL 300 python bench.py > gpurun_out/bench_line_v8.json 2> gpurun_out/bench_err.log; python -c "
import json; d=json.loads(open('gpurun_out/bench_line_v8.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
