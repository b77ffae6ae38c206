for cfg in "1 16" "1 32" "2 16" "2 32"; do
  set -- $cfg
  echo "== MF=$1 BK=$2"
  B2_CONTRACT_MF=$1 B2_CONTRACT_BK=$2 timeout 600 python -m pytest tests/test_gpu_config.py tests/test_gpu_contract.py tests/test_gpu_parity.py -m gpu -q -x -k "conv2d" 2>&1 | tail -1
  B2_CONTRACT_MF=$1 B2_CONTRACT_BK=$2 timeout 300 python scripts/bench_suite.py --only conv2d_bias --reps 10 --out gpurun_out/c.json 2>&1 | grep conv2d
done
