#!/bin/bash
# ncu --set full of the bucket and split kernels at N = 2^25 (C5 physics) with source,
# then the C5 and C4 launch lists.  usage: gpu_ncu_r3.sh TAG
TAG=${1:-r3}
O=gpurun_out/$TAG
mkdir -p $O
CMD="python bench.py --n 33554432 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > $O/plain_n2p25.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"bucket_kernel|split_kernel" -s 4 -c 2 -o $O/full_n2p25 -f $CMD > $O/ncu_full.log 2>&1
ncu -i $O/full_n2p25.ncu-rep --page raw --csv > $O/full_raw.csv 2>/dev/null
ncu -i $O/full_n2p25.ncu-rep --page source --csv --kernel-name regex:bucket_kernel --print-source cuda,sass > $O/bucket_src.csv 2>/dev/null
ncu -i $O/full_n2p25.ncu-rep --page source --csv --kernel-name regex:split_kernel --print-source cuda,sass > $O/split_src.csv 2>/dev/null
CMD2="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD2 > $O/plain_C5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_C5.csv $CMD2 > $O/ncu_launch.log 2>&1
CMD4="python bench.py --workload C4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD4 > $O/plain_C4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_C4.csv $CMD4 > $O/ncu_launch4.log 2>&1
echo done
