echo "256 thr BK32"; timeout 300 python scripts/probe_dgemm.py
echo "512 thr BK32"; B2_DGEMM_THREADS=512 timeout 300 python scripts/probe_dgemm.py
echo "512 thr BK16"; B2_DGEMM_THREADS=512 B2_DGEMM_BK=16 timeout 300 python scripts/probe_dgemm.py
B2_DGEMM_THREADS=512 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_config.py -m gpu -q -x -k "gemm or dgemm or matmul" 2>&1 | tail -1
