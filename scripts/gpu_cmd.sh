python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
B2_FORCE_SLAB=1 B2_SLAB_FORCE_SPLIT=1 timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/slab1.json 2> gpurun_out/slab1.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/slab1.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'])"
tail -3 gpurun_out/slab1.err
timeout -s KILL 600 python -m pytest tests/test_gpu_dist.py -q 2>&1 | tail -2
