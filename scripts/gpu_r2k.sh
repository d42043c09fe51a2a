#!/bin/bash
mkdir -p gpurun_out/r2k
for B1 in 7 8 9; do
RBM_B1=$B1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2k/bench_C5_b1_$B1.log 2>&1
done
RBM_B1=9 timeout 300 python bench.py --workload C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2k/bench_C4_b1_9.log 2>&1
timeout 300 python bench.py --workload C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2k/bench_C4.log 2>&1
