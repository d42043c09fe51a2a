#!/bin/bash
# one gpurun call: smoke, GPU parity tests, default bench, and the scatter design microbenchmark
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv >> gpurun_out/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo rc=$? >> gpurun_out/bench_default.log
MB=scripts/microbench/scatter_mb
timeout 300 $MB all > gpurun_out/mb_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum --clock-control none -k regex:"scatter|copy" --csv --log-file gpurun_out/mb_ncu.csv $MB all > gpurun_out/mb_ncu.log 2>&1
echo done
