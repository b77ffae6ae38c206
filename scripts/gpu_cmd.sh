python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for c in 4 0 2 8; do echo "== chunk $c"; B2_SMALL_RED_CHUNK=$c timeout -s KILL 300 python scripts/bench_suite.py --only nbody --out gpurun_out/nb.json 2>&1 | grep -E "ms "; done
timeout -s KILL 900 python -m pytest tests -q -m gpu -rf -o faulthandler_timeout=300 2>&1 | grep -E "FAILED|passed|failed|Error" | head -8
