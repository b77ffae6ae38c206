python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 200 python -m pytest tests/test_gpu_dist.py -q -x -o faulthandler_timeout=100 2>&1 | tail -2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555"
for env in "B2_SLAB_OVERLAP=0" "B2_SLAB_OVERLAP=1" "B2_SLAB_FORCE_SPLIT=1"; do
env B2_FORCE_SLAB=1 $env timeout -s KILL 200 $TR bench.py --steps 5 --warmup 3 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', d['ms_per_step'], d['config'])"
done
