#!/bin/bash
# RBM-r apply: single-increment fast path; ids per bucket 1024 / 512 / 256
mkdir -p gpurun_out/r2v
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_physics.py tests/test_cluster_gpu.py -k "rbmr or cluster or physics or m2" -q -rf -x > gpurun_out/r2v/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2v/t.log
B="timeout -s KILL 300 python bench.py --scheme rbmr --steps 16 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/r2v/w1024.log 2>&1
RBM_RBMR_W=512 $B > gpurun_out/r2v/w512.log 2>&1
RBM_RBMR_W=256 $B > gpurun_out/r2v/w256.log 2>&1
RBM_RBMR_W=512 timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -k "rbmr" -q -rf -x > gpurun_out/r2v/t512.log 2>&1
echo "rc=$?" >> gpurun_out/r2v/t512.log
