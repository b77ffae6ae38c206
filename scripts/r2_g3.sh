timeout 1800 python scripts/variant_survey.py 2>&1 | grep "^{"
