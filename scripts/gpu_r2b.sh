#!/bin/bash
# round 2: AoS-record kernels -- GPU tests, bench (C5 default, C4), phase profile
mkdir -p gpurun_out/r2b
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2b/bench_C5.log 2>&1
echo "rc=$?" >> gpurun_out/r2b/bench_C5.log
RBM_PHASE_PROF=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2b/bench_prof.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --maxfail=15 -x --durations=10 > gpurun_out/r2b/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b/gputest.log
timeout 300 python bench.py --workload C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2b/bench_C4.log 2>&1
