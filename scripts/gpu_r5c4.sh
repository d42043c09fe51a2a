#!/bin/bash
# --set full captures of the hot kernels of the BASELINE target config C4 (N = 1e8, p = 4:
# lane-group bucket kernel + splitter) at full size, of the C5 p = 8 bucket kernel at 2^25,
# and of the RBM-r emit / apply kernels at 2^25.   usage: gpu_r5c4.sh TAG
TAG=${1:-r5c4}
O=gpurun_out/$TAG
mkdir -p $O
F="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
cap() {  # name, kernel regex, skip, count, bench args...
  local name=$1 rx=$2 sk=$3 cn=$4; shift 4
  timeout 300 python bench.py "$@" $F > $O/plain_$name.log 2>&1 || return
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $sk -c $cn -o $O/prof_$name -f python bench.py "$@" $F > $O/ncu_$name.log 2>&1
  ncu -i $O/prof_$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
  ncu -i $O/prof_$name.ncu-rep --page source --csv --kernel-name regex:bucket_kernel --print-source cuda,sass > $O/${name}_bucket_src.csv 2>/dev/null
}
cap c4 "split_kernel|bucket_kernel" 4 2 --workload C4
cap c5p8 "bucket_kernel" 2 1 --p 8 --n 33554432
cap rbmr "rbmr_emit_kernel|rbmr_bucket_apply_kernel" 4 2 --scheme rbmr --n 33554432
rm -f $O/*.ncu-rep $O/*.ncu-rep.tmp
echo done
