./scripts/heatlab/heatlab 40 2>&1 | grep generated
./scripts/heatlab/heatlab 2500 2>&1 | grep generated
