#!/bin/bash
# RBM-r Jacobi without the per-step slot store: RBM-r tests, C5 RBM-r bench + launch list;
# one --set full capture of the C4 bucket kernel (source lines)
O=gpurun_out/r4b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cluster_gpu.py tests/test_partition_rbmr_gpu.py tests/test_rbmr_seq_gpu.py tests/test_checked_gpu.py -m gpu -q -p no:cacheprovider -rf -k "rbmr or cluster or sbm or checked" > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 300 python bench.py --scheme rbmr --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5rbmr.log 2>&1
CMDR="python bench.py --scheme rbmr --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_rbmr.csv $CMDR > $O/ncu_launch_rbmr.log 2>&1
CMD4="python bench.py --workload C4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bucket_kernel" -s 3 -c 1 -o $O/prof_c4 -f $CMD4 > $O/ncu_c4.log 2>&1
ncu -i $O/prof_c4.ncu-rep --page raw --csv > $O/c4_raw.csv 2>/dev/null
ncu -i $O/prof_c4.ncu-rep --page source --csv --kernel-name regex:bucket_kernel --print-source cuda,sass > $O/c4_bucket_src.csv 2>/dev/null
echo done
