#!/bin/bash
# layouts up to B = 20 on one GPU: N = 2^30 sampled parity; bench at 2^30 and 2^31 - 1
mkdir -p gpurun_out/r2z
free -g > gpurun_out/r2z/mem.txt
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py -k "full_size_sampled and C5max" -q -rf -x > gpurun_out/r2z/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2z/t.log
for N in 1073741824 2147483647; do
timeout -s KILL 600 python bench.py --n $N --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2z/n$N.log 2>&1
echo "rc=$?" >> gpurun_out/r2z/n$N.log
done
