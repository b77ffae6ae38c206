PAIR=1 ./scripts/heatlab/jaclab 400
