python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for n in 4096 8192 16384; do for p in 0 1; do for g in 4 8 16; do
echo "n=$n pair=$p group=$g $(B2_TC_PAIR=$p B2_TC_GROUP=$g timeout -s KILL 60 python scripts/probe_sgemm.py $n 3 2>&1 | tail -1)"
done; done; done
