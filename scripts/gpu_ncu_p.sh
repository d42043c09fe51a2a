#!/bin/bash
# ncu source-level capture of the bucket kernel at batch size P (default 8)
mkdir -p gpurun_out
P=${P:-8}
CMD="python bench.py --n 33554432 --p $P --steps 2 --warmup 2 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_p$P.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bucket_" -s 2 -c 1 -o gpurun_out/prof_p$P -f $CMD > gpurun_out/ncu_p$P.log 2>&1
echo done
