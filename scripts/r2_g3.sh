timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k softmax 2>&1 | tail -3
