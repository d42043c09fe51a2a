#!/bin/bash
# RBM-r' expected write counters (tags in the AoS padding word)
mkdir -p gpurun_out/r2r
timeout -s KILL 900 python -m pytest tests/test_rbmr_seq_gpu.py tests/test_cluster_gpu.py tests/test_gpu_parity.py -k "seq or rbmr or cluster or Seq" -q -rf -x > gpurun_out/r2r/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2r/t.log
timeout -s KILL 300 python bench.py --scheme rbmr_seq --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2r/bench_seq.log 2>&1
echo "rc=$?" >> gpurun_out/r2r/bench_seq.log
timeout -s KILL 300 python bench.py --scheme rbmr --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2r/bench_rbmr.log 2>&1
echo "rc=$?" >> gpurun_out/r2r/bench_rbmr.log
