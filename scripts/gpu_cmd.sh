python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for a in 1 0 1; do
  B2_ALIGN_TILES=$a timeout -s KILL 300 python scripts/bench_suite.py --only heat_3d,jacobi_2d,go_fast,softmax --out gpurun_out/align$a.json 2>&1 | grep -v "^\s*$" | tail -6
done
timeout -s KILL 900 python -m pytest tests -q -m gpu -x -o faulthandler_timeout=300 2>&1 | tail -3
