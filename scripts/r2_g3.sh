ncu --set full --clock-control none --import-source on -k regex:conv2d_bias_1 -c 1 -o gpurun_out/conv_slide60 python scripts/bench_suite.py --only conv2d_bias --reps 1 --out gpurun_out/s_conv_ncu.json > gpurun_out/ncu_conv.log 2>&1
tail -1 gpurun_out/ncu_conv.log
