#!/bin/bash
mkdir -p gpurun_out
RBM_PHASE_PROF=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_prof.log 2>&1
RBM_PHASE_PROF=1 RBM_BUCKET_TARGET=1024 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_prof1024.log 2>&1
echo done
