nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host.txt; nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv >> gpurun_out/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo rc=$? >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo rc=$? >> gpurun_out/bench_reference.log
for W in C1 C2 C3 C4; do timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$W.log 2>&1; done
for P in 8 32; do timeout 300 python bench.py --p $P --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5p$P.log 2>&1; done
timeout 300 python bench.py --scheme rbmr --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5rbmr.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C5.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python bench.py --n 33554432 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline"
timeout 300 $CMD2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bucket_pair|scatter" -s 4 -c 2 -o gpurun_out/prof_r1_final -f $CMD2 > gpurun_out/ncu_full.log 2>&1
