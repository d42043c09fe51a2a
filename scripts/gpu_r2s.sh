#!/bin/bash
# 24-byte RBM-r increment records (fp32 d=3); RBM-r' tests incl. the 2^21 fp32 determinism case
mkdir -p gpurun_out/r2s
timeout -s KILL 900 python -m pytest tests/test_rbmr_seq_gpu.py tests/test_cluster_gpu.py tests/test_partition_rbmr_gpu.py tests/test_gpu_physics.py tests/test_gpu_parity.py -k "seq or rbmr or cluster or Seq or physics or m2" -q -rf -x > gpurun_out/r2s/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2s/t.log
timeout -s KILL 300 python bench.py --scheme rbmr_seq --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2s/bench_seq.log 2>&1
echo "rc=$?" >> gpurun_out/r2s/bench_seq.log
timeout -s KILL 300 python bench.py --scheme rbmr --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2s/bench_rbmr.log 2>&1
echo "rc=$?" >> gpurun_out/r2s/bench_rbmr.log
