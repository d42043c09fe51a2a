#!/bin/bash
mkdir -p gpurun_out/r2f
timeout 1200 python -m pytest tests/test_cluster_gpu.py tests/test_partition_procs_gpu.py -q -rf -s > gpurun_out/r2f/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2f/t.log
