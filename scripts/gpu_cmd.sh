python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
P="python scripts/probe_time.py"
for w in gemver atax bicg; do
  if [ $w = gemver ]; then S='{"N": 8000}'; else S='{"M": 8000, "N": 8000}'; fi
  $P $w.raw "$S" 3 > gpurun_out/plain_$w.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l_$w.csv $P $w.raw "$S" 3 > gpurun_out/ncu_$w.log 2>&1
  tail -4 gpurun_out/plain_$w.log
done
