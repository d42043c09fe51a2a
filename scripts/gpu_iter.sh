#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_wealth_gpu.py -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_wealth.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_wealth.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --workload wealth --steps 3000 --warmup 10 --no-cpu-baseline > gpurun_out/bench_wealth.log 2>&1
timeout 300 python bench.py --workload wealth --n 100000000 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_wealth_1e8.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_default.log 2>&1
echo done
