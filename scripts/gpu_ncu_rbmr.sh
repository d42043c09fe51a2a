#!/bin/bash
# ncu --set full of the RBM-r kernels at N = 2^25 (C5 physics)
O=gpurun_out/${1:-r3nr}
mkdir -p $O
CMD="python bench.py --scheme rbmr --n 33554432 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"rbmr_emit|rbmr_bucket_apply" -s 2 -c 2 -o $O/rbmr_full -f $CMD > $O/ncu_full.log 2>&1
ncu -i $O/rbmr_full.ncu-rep --page raw --csv > $O/full_raw.csv 2>/dev/null
ncu -i $O/rbmr_full.ncu-rep --page source --csv --kernel-name regex:rbmr_bucket_apply --print-source cuda,sass > $O/apply_src.csv 2>/dev/null
ncu -i $O/rbmr_full.ncu-rep --page source --csv --kernel-name regex:rbmr_emit --print-source cuda,sass > $O/emit_src.csv 2>/dev/null
echo done
