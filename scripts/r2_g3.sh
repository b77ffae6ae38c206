timeout 900 python -m pytest tests -m gpu -q -x -k "atax or bicg or mvt or gesummv or gemver or azimint" 2>&1 | tail -3
timeout 600 python scripts/variant_survey.py atax,bicg,mvt,gesummv,gemver 2>&1 | grep "^{"
