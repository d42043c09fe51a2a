#!/bin/bash
mkdir -p gpurun_out/r2g
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "two_pass or full_size or permutation or oversized or c2_configured or step_vs_run or determinism" > gpurun_out/r2g/par.log 2>&1
echo "rc=$?" >> gpurun_out/r2g/par.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2g/bench_C5.log 2>&1
RBM_FUSED=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2g/bench_C5_unfused.log 2>&1
timeout 300 python bench.py --workload C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2g/bench_C4.log 2>&1
timeout 300 python bench.py --p 8 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2g/bench_p8.log 2>&1
