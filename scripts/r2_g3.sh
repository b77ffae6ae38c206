timeout 300 python scripts/probe_dgemm.py
timeout 1200 python -m pytest tests -m gpu -q -x -k "gemm or matmul or summa or k2mm or k3mm or dgemm or doitgen or config" 2>&1 | tail -3
