#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --n 33554432 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bucket_pair" -s 2 -c 1 -o gpurun_out/prof_src5 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo done
