#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_default.log 2>&1; echo rc=$? >> gpurun_out/bench_default.log
for T in 1024 1280 1536; do RBM_BUCKET_TARGET=$T timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_t$T.log 2>&1; done
RBM_SPLIT_CFG=small timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_small.log 2>&1
echo done
