timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline'])"
timeout 1800 python scripts/bench_suite.py --reps 10 --out gpurun_out/bench_suite_r02d.json > gpurun_out/f_suite_d.log 2>&1; tail -12 gpurun_out/f_suite_d.log
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_suite_r02d.json"))
for k, x in d.items():
    print(k, round(x["ms_per_run"], 4), x.get("roofline") and round(x["roofline"]["frac"], 3), round(x.get("step_share_top") or 0, 3), x.get("kernel_time_basis"))
PY
