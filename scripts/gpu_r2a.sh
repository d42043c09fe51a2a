#!/bin/bash
# round 2, first check: the new parity/long-run/ensemble tests on the round-1 kernels + bench
mkdir -p gpurun_out/r2a
nvidia-smi > gpurun_out/r2a/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=30 > gpurun_out/r2a/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a/gputest.log
timeout 600 python bench.py > gpurun_out/r2a/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2a/bench.log
