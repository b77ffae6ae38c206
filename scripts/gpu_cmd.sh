python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for cfg in 1 0; do
  echo "== EAGER_LOGIC=$cfg"
  B2_EAGER_LOGIC=$cfg timeout -s KILL 300 python scripts/bench_suite.py --only azimint_naive,go_fast,nbody --out gpurun_out/el_$cfg.json 2>&1 | grep -E "ms " | tail -4
done
timeout -s KILL 900 python -m pytest tests -q -m gpu -x -o faulthandler_timeout=300 2>&1 | tail -3
