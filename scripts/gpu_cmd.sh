python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
run() { echo "== $*"; env "$@" timeout -s KILL 300 python scripts/bench_suite.py --only jacobi_2d,go_fast,softmax --reps 10 --out gpurun_out/j.json 2>&1 | grep -E "ms "; }
run B2_TILE_BY=8
run B2_TILE_BY=4
run B2_TILE_BY=16
run B2_TILE_BY=32
run B2_TILE_BY=16 B2_VEC=1
run B2_TILE_BY=8 B2_VEC=1
