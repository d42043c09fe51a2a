#!/bin/bash
# launch lists (time + DRAM bytes) of the RBM-r and RBM-r' steps at C5, and one --set full
# capture of the RBM-r' sweep and link kernels at N = 2^25
mkdir -p gpurun_out/r2aa
O=gpurun_out/r2aa
for S in rbmr rbmr_seq; do
CMD="python bench.py --scheme $S --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > $O/plain_$S.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none -c 60 --csv --log-file $O/launches_$S.csv $CMD > $O/ncu_$S.log 2>&1
done
CMD2="python bench.py --scheme rbmr_seq --n 33554432 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD2 > $O/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rbmr_seq_dep|rbmr_bucket_apply" -s 2 -c 2 -o $O/seq_full -f $CMD2 > $O/ncu_full.log 2>&1
echo done
