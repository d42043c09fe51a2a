#!/bin/bash
# smaller buckets (mean 1024, B = 18) with 160-thread CTAs (up to 6 CTAs per SM) vs the default
mkdir -p gpurun_out/r2u
B="timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
RBM_LIB=paper_1812_10575_b200/librbm_bk160.so RBM_BUCKET_TARGET=1024 $B > gpurun_out/r2u/t1024_b9.log 2>&1
RBM_LIB=paper_1812_10575_b200/librbm_bk160.so RBM_BUCKET_TARGET=1024 RBM_B1=8 $B > gpurun_out/r2u/t1024_b8.log 2>&1
RBM_LIB=paper_1812_10575_b200/librbm_bk160.so RBM_BUCKET_TARGET=1024 RBM_B1=10 $B > gpurun_out/r2u/t1024_b10.log 2>&1
RBM_LIB=paper_1812_10575_b200/librbm_bk160.so RBM_BUCKET_TARGET=1024 $B --workload C4 > gpurun_out/r2u/C4_t1024.log 2>&1
$B > gpurun_out/r2u/base.log 2>&1
