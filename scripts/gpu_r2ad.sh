#!/bin/bash
# --set full capture of the C4 bucket kernel (p = 4 lane groups, keyed f32 d=2 records) at N = 2^25
mkdir -p gpurun_out/r2ad
O=gpurun_out/r2ad
CMD="python bench.py --workload C4 --n 33554432 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bucket_kernel|split_kernel" -s 4 -c 2 -o $O/c4_full -f $CMD > $O/ncu_full.log 2>&1
echo done
