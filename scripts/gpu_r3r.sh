#!/bin/bash
# RBM-r: 16-byte increment records, canonical summation order; tests + bench
O=gpurun_out/${1:-r3r}
mkdir -p $O
timeout 300 python bench.py --scheme rbmr --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5rbmr.log 2>&1
timeout 300 python bench.py --scheme rbmr_seq --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5rbmr_seq.log 2>&1
timeout 1500 python -m pytest tests -m gpu -k "rbmr or cluster or physics or partition_rbmr" -q -x -rf -p no:cacheprovider > $O/t.log 2>&1; echo rc=$? >> $O/t.log
echo done
