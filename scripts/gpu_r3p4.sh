#!/bin/bash
O=gpurun_out/${1:-r3p4}
mkdir -p $O
RBM_PHASE_PROF=1 timeout 300 python bench.py --workload C4 --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > $O/prof_c4.log 2>&1
CMD="python bench.py --workload C4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"bucket_kernel" -s 2 -c 1 -o $O/c4_full -f $CMD > $O/ncu_full.log 2>&1
ncu -i $O/c4_full.ncu-rep --page raw --csv > $O/full_raw.csv 2>/dev/null
ncu -i $O/c4_full.ncu-rep --page source --csv --kernel-name regex:bucket_kernel --print-source cuda,sass > $O/bucket_src.csv 2>/dev/null
echo done
