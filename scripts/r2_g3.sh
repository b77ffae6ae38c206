timeout 900 python -m pytest tests/test_gpu_contract.py -q -x 2>&1 | tail -2
timeout 3000 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python scripts/variant_survey.py doitgen 2>&1 | grep "^{"
