#!/bin/bash
# dev tool: build, GPU tests, BLAS-2 timings, launch list + ncu of the top kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
for w in 'gemver.raw {"N":8000}' 'atax.raw {"M":8000,"N":8000}' 'bicg.raw {"N":8000,"M":8000}'; do
  set -- $w; python scripts/probe_time.py $1 "$2" 4 2>&1 | tail -2
done
python bench.py --steps 2 --warmup 1 > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launches.log 2>&1
python scripts/probe_time.py heat_3d.raw '{"N": 400, "TSTEPS": 3}' 2 > gpurun_out/plain_heat.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:b2_map -s 2 -c 1 -o gpurun_out/prof_heat python scripts/probe_time.py heat_3d.raw '{"N": 400, "TSTEPS": 3}' 2 > gpurun_out/ncu_heat.log 2>&1
python scripts/probe_time.py bicg.raw '{"N": 8000, "M": 8000}' 2 > gpurun_out/plain_bicg.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:b2_rp -s 1 -c 1 -o gpurun_out/prof_bicg python scripts/probe_time.py bicg.raw '{"N": 8000, "M": 8000}' 2 > gpurun_out/ncu_bicg.log 2>&1
echo done
