python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
run() { echo "== $*"; env "$@" timeout -s KILL 300 python scripts/bench_suite.py --only heat_3d --reps 10 --out gpurun_out/pf.json 2>&1 | grep -E "ms " | tail -1; }
for i in 1 2; do
run B2_MARCH_BX=64
run B2_MARCH_BX=64 B2_VEC=12
run B2_MARCH_BX=128 B2_MARCH_BY=4
run B2_MARCH_BX=32 B2_MARCH_BY=16
done
