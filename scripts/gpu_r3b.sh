#!/bin/bash
# microbenchmarks: output-stage staging vs direct stores; per-record random scatter sweep
O=gpurun_out/r3b
mkdir -p $O
timeout 120 ./scripts/microbench/runs_mb > $O/runs_mb.log 2>&1
timeout 300 ./scripts/microbench/scatter_mb a > $O/scatter_mb.log 2>&1
echo done
