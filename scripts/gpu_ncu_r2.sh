#!/bin/bash
# ncu --set full of the bucket and split kernels at N = 2^25 (C5 physics), plus the C5 launch list
# usage: gpu_ncu_r2.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out/$TAG
CMD="python bench.py --n 33554432 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/$TAG/plain_n2p25.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"bucket_kernel|split_kernel" -s 4 -c 2 -o gpurun_out/$TAG/full_n2p25 -f $CMD > gpurun_out/$TAG/ncu_full.log 2>&1
CMD2="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD2 > gpurun_out/$TAG/plain_C5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/$TAG/launches_C5.csv $CMD2 > gpurun_out/$TAG/ncu_launch.log 2>&1
echo done
