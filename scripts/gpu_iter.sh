#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_rbmr_seq_gpu.py -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_seq.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_seq.log
timeout 300 python bench.py --scheme rbmr_seq --n 16777216 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_seq.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_default.log 2>&1
echo done
