#!/bin/bash
# every config with the CPU oracle baseline beside it,
# plus the C4 launch list (DRAM bytes per kernel launch).
mkdir -p gpurun_out/bt
O=gpurun_out/bt
for W in C1 C2 C3 C4; do timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-e2e > $O/bench_$W.log 2>&1; done
CMD="python bench.py --workload C4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > $O/plain_C4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/launches_C4.csv $CMD > $O/ncu_C4.log 2>&1
echo done
