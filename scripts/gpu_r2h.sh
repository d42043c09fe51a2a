#!/bin/bash
mkdir -p gpurun_out/r2h
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_physics.py tests/test_partition_rbmr_gpu.py tests/test_cluster_gpu.py tests/test_rbmr_seq_gpu.py -q -rf -k "rbmr or cluster or sbm or RBM" > gpurun_out/r2h/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2h/t.log
timeout 300 python bench.py --scheme rbmr --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2h/bench_rbmr.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2h/bench_C5.log 2>&1
