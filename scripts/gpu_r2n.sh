#!/bin/bash
# RBM-r' sweep with acquire/release flags and the p = 2 pair path
mkdir -p gpurun_out/r2n
timeout -s KILL 600 python -m pytest tests/test_rbmr_seq_gpu.py tests/test_cluster_gpu.py -q -rf -x > gpurun_out/r2n/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2n/t.log
timeout -s KILL 300 python bench.py --scheme rbmr_seq --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2n/bench_seq.log 2>&1
echo "rc=$?" >> gpurun_out/r2n/bench_seq.log
