#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_partition_gpu.py -q --timeout 600 -p no:cacheprovider -rf -x > gpurun_out/pytest_part.log 2>&1; echo rc=$? >> gpurun_out/pytest_part.log
CMD2="python bench.py --n 33554432 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline"
timeout 300 $CMD2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bucket_pair|scatter_kernel" -s 4 -c 2 -o gpurun_out/prof_src -f $CMD2 > gpurun_out/ncu_full.log 2>&1
echo done
