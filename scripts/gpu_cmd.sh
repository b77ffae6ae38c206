python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555"
timeout -s KILL 300 python bench.py 2>&1 | grep metric | cut -c1-3000
timeout -s KILL 300 python bench.py --workload jacobi_2d 2>&1 | grep metric | cut -c1-3000
timeout -s KILL 300 python bench.py --impl reference 2>&1 | grep metric | cut -c1-600
timeout -s KILL 300 $TR bench.py --gpus 1 2>&1 | grep metric | cut -c1-2000
B2_FORCE_SLAB=1 timeout -s KILL 300 $TR bench.py --gpus 1 --workload jacobi_2d 2>&1 | grep metric | cut -c1-2000
