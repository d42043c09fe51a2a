#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x -k "rbmr or determinism or replicas" > gpurun_out/pytest_rbmr.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_rbmr.log
timeout 300 python bench.py --scheme rbmr --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5rbmr.log 2>&1
timeout 300 python bench.py --direct --workload C5 --steps 5 --warmup 2 > gpurun_out/bench_direct.log 2>&1
timeout 300 python bench.py --direct --workload C5 --n 16384 --steps 20 --warmup 2 > gpurun_out/bench_direct16k.log 2>&1
echo done
