#!/bin/bash
mkdir -p gpurun_out/r2e
timeout 1200 python -m pytest tests/test_partition_rbmr_gpu.py tests/test_partition_gpu.py tests/test_partition_procs_gpu.py -q -rf -x > gpurun_out/r2e/part.log 2>&1
echo "rc=$?" >> gpurun_out/r2e/part.log
