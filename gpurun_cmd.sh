timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -s -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
CMD="python bench.py --n 16777216 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bucket_step|scatter_kernel" -s 3 -c 3 -o gpurun_out/prof_r1b -f $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$? >> gpurun_out/ncu_full.log
timeout 900 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -s -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_full.log
