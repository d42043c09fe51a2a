#!/bin/bash
# A/B: default librbm.so vs a design variant (RBM_LIB), C5 and C4 bench lines
O=gpurun_out/${1:-r3v}; V=$2
mkdir -p $O
for L in librbm.so $V; do
  RBM_LIB=$PWD/paper_1812_10575_b200/$L timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5_$L.log 2>&1
  RBM_LIB=$PWD/paper_1812_10575_b200/$L timeout 300 python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4_$L.log 2>&1
done
echo done
