./scripts/heatlab/heatlab 2500 2>&1
