#!/bin/bash
# largest single-GPU systems: N = 2^29 and 2^30 (layout limits)
mkdir -p gpurun_out/r2y
for N in 536870912 1073741824; do
timeout -s KILL 600 python bench.py --n $N --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2y/n$N.log 2>&1
echo "rc=$?" >> gpurun_out/r2y/n$N.log
done
