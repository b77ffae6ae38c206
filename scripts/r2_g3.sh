timeout 3000 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python scripts/variant_survey.py adi,jacobi_2d,heat_3d,jacobi_1d,softmax 2>&1 | grep "^{"
