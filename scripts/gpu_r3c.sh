#!/bin/bash
# warp-specialized pass-2 splitter: perf + the tests that run the 2-pass layouts
O=gpurun_out/${1:-r3c}
mkdir -p $O
RBM_PHASE_PROF=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > $O/prof_c5.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.log 2>&1
timeout 300 python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4.log 2>&1
timeout 300 python bench.py --scheme rbmr --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5rbmr.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_partition_gpu.py tests/test_partition_rbmr_gpu.py tests/test_rbmr_seq_gpu.py tests/test_gpu_longrun.py -q -x -rf -p no:cacheprovider > $O/t.log 2>&1; echo rc=$? >> $O/t.log
echo done
