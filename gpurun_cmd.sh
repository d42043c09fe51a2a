timeout 900 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
for cfg in "1024 9" "2048 8" "2048 9"; do set -- $cfg; RBM_BUCKET_TARGET=$1 RBM_B1=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$1_$2.log 2>&1; done
