#!/bin/bash
# Round-2 (session 2) record: smoke, every -m gpu test, bench lines for every workload,
# reference arm, ncu launch lists (C5, C4) and one --set full capture of the
# two hot kernels (split, bucket step) at N = 2^25.   usage: gpu_full_r2.sh TAG
TAG=${1:-r4full}
O=gpurun_out/$TAG
mkdir -p $O
nproc > $O/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/host.txt; nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv >> $O/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo pytest_rc=$? >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo rc=$? >> $O/bench_default.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.log 2>&1; echo rc=$? >> $O/bench_reference.log
for W in C1 C2 C3 C4; do timeout 300 python bench.py --workload $W --steps 20 --warmup 3 > $O/bench_$W.log 2>&1; done
timeout 300 python bench.py --workload C1 --steps 1000 --warmup 10 --no-cpu-baseline > $O/bench_C1_1000.log 2>&1
for P in 8 32; do timeout 300 python bench.py --p $P --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5p$P.log 2>&1; done
timeout 300 python bench.py --scheme rbmr --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5rbmr.log 2>&1
timeout 300 python bench.py --scheme rbmr_seq --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5rbmr_seq.log 2>&1
timeout 300 python bench.py --workload wealth --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_wealth.log 2>&1
timeout 300 python bench.py --direct --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_direct.log 2>&1
timeout 300 python bench.py --workload verlet --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_verlet.log 2>&1
timeout 300 python bench.py --workload opinion --steps 1000 --warmup 10 --no-cpu-baseline > $O/bench_opinion.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_C5.csv $CMD > $O/ncu_launch.log 2>&1
CMD4="python bench.py --workload C4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD4 > $O/plain4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_C4.csv $CMD4 > $O/ncu_launch4.log 2>&1
CMD2="python bench.py --n 33554432 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD2 > $O/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"split_kernel|bucket_kernel" -s 4 -c 2 -o $O/prof_full -f $CMD2 > $O/ncu_full.log 2>&1
echo done
# RBM-r kernels at N = 2^25 (--set full) and the RBM-r launch lists at C5
CMDR="python bench.py --scheme rbmr --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMDR > $O/plain_rbmr.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_rbmr.csv $CMDR > $O/ncu_launch_rbmr.log 2>&1
ncu -i $O/prof_full.ncu-rep --page raw --csv > $O/full_raw.csv 2>/dev/null
ncu -i $O/prof_full.ncu-rep --page source --csv --kernel-name regex:bucket_kernel --print-source cuda,sass > $O/bucket_src.csv 2>/dev/null
ncu -i $O/prof_full.ncu-rep --page source --csv --kernel-name regex:split_kernel --print-source cuda,sass > $O/split_src.csv 2>/dev/null
echo done2
