#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_direct_gpu.py -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_direct.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_direct.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
echo done
