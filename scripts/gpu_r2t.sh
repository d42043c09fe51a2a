#!/bin/bash
# occupancy sensitivity of the bucket kernel (3 -> 2 -> 1 CTAs per SM via padded smem): the
# evidence for the cluster (on-chip pass 2) evaluation in DESIGN.md section 8
mkdir -p gpurun_out/r2t
B="timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/r2t/cta3.log 2>&1
RBM_BUCKET_SMEM_MIN=100000 $B > gpurun_out/r2t/cta2.log 2>&1
RBM_BUCKET_SMEM_MIN=150000 $B > gpurun_out/r2t/cta1.log 2>&1
