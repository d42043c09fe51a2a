#!/bin/bash
mkdir -p gpurun_out/r2i
timeout 1200 python -m pytest tests/test_verlet_gpu.py tests/test_gpu_parity.py tests/test_partition_gpu.py -q -rf -x -k "verlet or Verlet or two_pass or c2 or sphere or 100_steps or one_step_parity or bit_identical" > gpurun_out/r2i/t.log 2>&1
echo "rc=$?" >> gpurun_out/r2i/t.log
timeout 300 python bench.py --workload verlet --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2i/bench_verlet.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2i/bench_C5.log 2>&1
RBM_LIB=paper_1812_10575_b200/librbm_b256.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2i/bench_C5_b256.log 2>&1
RBM_LIB=paper_1812_10575_b200/librbm_b256.so timeout 300 python bench.py --workload C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2i/bench_C4_b256.log 2>&1
timeout 300 python bench.py --workload C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2i/bench_C4.log 2>&1
