#!/bin/bash
# quick perf check: phase profile run + default bench (no tests)
mkdir -p gpurun_out
RBM_PHASE_PROF=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_prof.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_default.log 2>&1
echo done
