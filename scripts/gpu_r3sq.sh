#!/bin/bash
# RBM-r' sweep: CTAs per SM sweep (RBM_SEQ_CTAS)
O=gpurun_out/${1:-r3sq}
mkdir -p $O
for S in 16 12 8 6 4 2; do
  RBM_SEQ_CTAS=$S timeout 300 python bench.py --scheme rbmr_seq --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/seq_$S.log 2>&1
done
echo done
