#!/bin/bash
# compile-time lane-group sizes: C4 (p=4), C5 p=8 / p=32 + the group-mode parity tests
O=gpurun_out/${1:-r3g}
mkdir -p $O
timeout 300 python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4.log 2>&1
for P in 8 32; do timeout 300 python bench.py --p $P --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5p$P.log 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_longrun.py tests/test_partition_gpu.py tests/test_gpu_physics.py -q -x -rf -p no:cacheprovider > $O/t.log 2>&1; echo rc=$? >> $O/t.log
echo done
