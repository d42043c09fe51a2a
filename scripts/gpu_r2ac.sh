#!/bin/bash
# RBM-r' sweep at 32 registers (16 CTAs x 4 warps per SM)
mkdir -p gpurun_out/r2ac
timeout -s KILL 900 python -m pytest tests/test_rbmr_seq_gpu.py tests/test_cluster_gpu.py -q -rf -x > gpurun_out/r2ac/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2ac/t.log
timeout -s KILL 300 python bench.py --scheme rbmr_seq --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2ac/seq.log 2>&1
