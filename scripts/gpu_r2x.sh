#!/bin/bash
# split smem header padding fix: RBM-r / RBM-r' at the B = 20 layout; RBM-r ids-per-bucket sweep
mkdir -p gpurun_out/r2x
timeout -s KILL 900 python -m pytest tests/test_rbmr_seq_gpu.py -q -rf -x > gpurun_out/r2x/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2x/t.log
B="timeout -s KILL 300 python bench.py --scheme rbmr --steps 16 --warmup 3 --no-cpu-baseline --no-e2e"
RBM_RBMR_W=256 $B > gpurun_out/r2x/w256.log 2>&1
RBM_RBMR_W=128 $B > gpurun_out/r2x/w128.log 2>&1
