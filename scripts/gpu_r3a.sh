#!/bin/bash
# session re-entry baseline: smoke, every -m gpu test, phase profile, C5 / C4 bench
O=gpurun_out/r3a
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
RBM_PHASE_PROF=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > $O/prof_c5.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.log 2>&1
timeout 300 python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo pytest_rc=$? >> $O/pytest_gpu.log
echo done
