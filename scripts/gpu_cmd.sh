python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python scripts/summa_projection.py f32 2>&1 | grep f32
nvidia-smi --query-gpu=clocks.sm,temperature.gpu,power.draw --format=csv
