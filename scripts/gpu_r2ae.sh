#!/bin/bash
# C4: fp32 Gaussian kernel through MUFU exp2, batch prefactors from host constants
mkdir -p gpurun_out/r2ae
O=gpurun_out/r2ae
timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_longrun.py tests/test_partition_gpu.py -q -rf -x > $O/t.log 2>&1
echo "rc=$?" >> $O/t.log
timeout -s KILL 300 python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4.log 2>&1
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.log 2>&1
timeout -s KILL 300 python bench.py --p 8 --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5p8.log 2>&1
