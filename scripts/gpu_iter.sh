#!/bin/bash
mkdir -p gpurun_out
RBM_PAIR_KERNEL=pair3 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_pair3.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_default.log 2>&1
RBM_PAIR_KERNEL=pair3 timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x > gpurun_out/pytest_pair3.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_pair3.log
echo done
