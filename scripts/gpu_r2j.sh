#!/bin/bash
mkdir -p gpurun_out/r2j
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_partition_gpu.py tests/test_verlet_gpu.py -q -rf -x -k "two_pass or c2 or 100_steps or bit_identical or permutation or full_size or verlet_steps" > gpurun_out/r2j/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2j/t.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2j/bench_C5.log 2>&1
timeout 300 python bench.py --workload C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2j/bench_C4.log 2>&1
timeout 300 python bench.py --scheme rbmr --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2j/bench_rbmr.log 2>&1
RBM_PHASE_PROF=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2j/bench_prof.log 2>&1
