#!/bin/bash
# split-kernel occupancy variants (A: 2 x 512-thread CTAs, 32 KB stages; D: 2 x 1024) + RBM-r' sweep profile
mkdir -p gpurun_out/r2m
B="timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/r2m/base.log 2>&1
RBM_LIB=paper_1812_10575_b200/librbm_spA.so $B > gpurun_out/r2m/spA.log 2>&1
RBM_LIB=paper_1812_10575_b200/librbm_spD.so $B > gpurun_out/r2m/spD.log 2>&1
RBM_LIB=paper_1812_10575_b200/librbm_spA.so $B --workload C4 > gpurun_out/r2m/spA_C4.log 2>&1
$B --workload C4 > gpurun_out/r2m/base_C4.log 2>&1
RBM_LIB=paper_1812_10575_b200/librbm_spA.so $B --scheme rbmr > gpurun_out/r2m/spA_rbmr.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none -k regex:rbmr_seq_dep -c 1 -o gpurun_out/r2m/seq_full \
  python bench.py --scheme rbmr_seq --n 16777216 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2m/ncu_seq.log 2>&1
echo rc=$? >> gpurun_out/r2m/ncu_seq.log
