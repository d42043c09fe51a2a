#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_verlet_gpu.py -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_verlet.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_verlet.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_default.log 2>&1
echo done
