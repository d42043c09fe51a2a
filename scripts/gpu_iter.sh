#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_opinion_gpu.py -q --timeout 600 -p no:cacheprovider -rf > gpurun_out/pytest_opinion.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_opinion.log
echo done
