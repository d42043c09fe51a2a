#!/bin/bash
# quick check: C5 / C4 bench lines + phase profile + the permutation / parity tests
O=gpurun_out/${1:-r3q}
mkdir -p $O
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.log 2>&1
timeout 300 python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4.log 2>&1
RBM_PHASE_PROF=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > $O/prof_c5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf -p no:cacheprovider > $O/t.log 2>&1; echo rc=$? >> $O/t.log
echo done
