#!/bin/bash
mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests/test_partition_procs_gpu.py tests/test_ensemble_gpu.py -q -rf -x > gpurun_out/r2c/procs.log 2>&1
echo "rc=$?" >> gpurun_out/r2c/procs.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c/bench_C5.log 2>&1
