#!/bin/bash
mkdir -p gpurun_out/r2d
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2d/bench_C5.log 2>&1
RBM_PHASE_PROF=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d/bench_prof.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --maxfail=10 --durations=5 > gpurun_out/r2d/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2d/gputest.log
timeout 300 python bench.py --workload C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2d/bench_C4.log 2>&1
timeout 300 python bench.py --p 8 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2d/bench_p8.log 2>&1
timeout 300 python bench.py --p 32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2d/bench_p32.log 2>&1
timeout 300 python bench.py --scheme rbmr --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d/bench_rbmr.log 2>&1
