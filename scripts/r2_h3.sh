#!/bin/bash
# rowred next-row L2 prefetch (B2_ROWRED_PF): timing A/B on softmax and the
# expanded-GEMV row dots, then the GPU parity tests with it on.
P="python scripts/probe_time.py"
S='{"N": 64, "H": 16, "SM": 512}'
A='{"M": 4000, "N": 4000}'
for r in 1 2; do
for pf in 0 1; do
  echo "== softmax pf=$pf"; B2_ROWRED_PF=$pf timeout 300 $P softmax.raw "$S" 20 2>&1 | tail -2
  echo "== atax.auto pf=$pf"; B2_ROWRED_PF=$pf timeout 300 $P atax.auto "$A" 20 2>&1 | tail -2
done; done
B2_ROWRED_PF=1 timeout 1200 python -m pytest tests -m gpu -x -q -k "softmax or atax or bicg or mvt or gesummv or rowred" 2>&1 | tail -3
