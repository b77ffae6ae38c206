timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -x 2>&1 | grep -E "^E |passed|failed" | head -20
timeout 600 python bench.py --workload matmul_f32 --steps 10 --warmup 3 2>&1 | tail -2 | cut -c1-1500
timeout 900 python bench.py --workload matmul --steps 3 --warmup 2 2>&1 | tail -2 | cut -c1-1500
