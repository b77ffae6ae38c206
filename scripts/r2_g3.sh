echo "== old (non-persistent) =="
timeout 600 python -c "
import runpy, sys
sys.path.insert(0, '.')
from paper_2107_00555_b200 import runtime as rt
rt._lib = rt.load_library('scripts/libb2_old.so')
sys.argv = ['x', 'f32']
runpy.run_path('scripts/summa_projection.py', run_name='__main__')" 2>&1 | tail -3
echo "== new (auto) =="
timeout 600 python scripts/summa_projection.py f32 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "f32 or sgemm or tf32 or presplit or tc" 2>&1 | tail -1
