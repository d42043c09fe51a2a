#!/bin/bash
# every -m gpu test + smoke
O=gpurun_out/${1:-r3full}
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo pytest_rc=$? >> $O/pytest_gpu.log
echo done
