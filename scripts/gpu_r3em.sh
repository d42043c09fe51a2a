#!/bin/bash
# RBM-r emit: CTAs per SM sweep through the smem-padding knob
O=gpurun_out/${1:-r3em}
mkdir -p $O
for S in 0 60000 77000 115000; do
  RBM_EMIT_SMEM=$S timeout 300 python bench.py --scheme rbmr --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > $O/emit_$S.log 2>&1
done
echo done
