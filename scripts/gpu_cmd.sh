python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for cfg in "8 16 1" "8 16 0" "16 16 1" "4 16 1" "8 24 1" "8 32 1" "4 32 1"; do
  set -- $cfg
  echo "== BY $1 vec $2 full $3"
  B2_MARCH_BY=$1 B2_VEC=$2 B2_FULL_TILES=$3 timeout -s KILL 120 python scripts/probe_time.py heat_3d.raw '{"N":400,"TSTEPS":20}' 2 2>&1 | grep -E "kernel|Error" | head -1
done
