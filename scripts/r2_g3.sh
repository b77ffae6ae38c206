timeout 1500 python -m pytest tests -m gpu -q -x -k "go_fast or softmax or fig4 or edges or region or parity" 2>&1 | tail -2
timeout 600 python scripts/variant_survey.py go_fast,softmax,fig4_loop 2>&1 | grep "^{"
