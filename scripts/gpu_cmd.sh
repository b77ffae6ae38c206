python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -k "atax or bicg or gemver or mvt or gesummv or rowpass" -o faulthandler_timeout=100 2>&1 | tail -1
for w in 'gemver.raw {"N":8000}' 'atax.raw {"M":8000,"N":8000}' 'bicg.raw {"N":8000,"M":8000}'; do
  set -- $w; echo "$1"; timeout -s KILL 120 python scripts/probe_time.py $1 "$2" 4 2>&1 | grep -E "rep 3|kernel|Error" | head -4
done
