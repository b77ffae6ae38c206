PAIR=1 timeout 300 ./scripts/heatlab/heatlab 40 2>&1
PAIR=1 timeout 300 ./scripts/heatlab/heatlab 1200 2>&1
