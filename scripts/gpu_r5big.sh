#!/bin/bash
# Larger final buckets (mean 4096) with 512-thread bucket CTAs, two per SM
# (build.py -DRBM_BUCKET_BLOCK=512 -DRBM_BUCKET_ITEMS=10 -DRBM_FUSED_CAP_MAX=8192 -o librbm_b512.so)
TAG=${1:-r5big}
O=gpurun_out/$TAG
mkdir -p $O
B="--steps 16 --warmup 3 --no-cpu-baseline --no-e2e"
for LIB in b512 b384; do
export RBM_LIB=$PWD/paper_1812_10575_b200/librbm_$LIB.so
[ -f $RBM_LIB ] || continue
for T in 4096 2048; do
  RBM_BUCKET_TARGET=$T timeout 300 python bench.py $B > $O/${LIB}_C5_t$T.log 2>&1
  RBM_BUCKET_TARGET=$T timeout 300 python bench.py --workload C4 $B > $O/${LIB}_C4_t$T.log 2>&1
  RBM_BUCKET_TARGET=$T timeout 300 python bench.py --p 8 $B > $O/${LIB}_C5p8_t$T.log 2>&1
done
RBM_BUCKET_TARGET=4096 RBM_B1=7 timeout 300 python bench.py $B > $O/${LIB}_C5_t4096_b1_7.log 2>&1
RBM_BUCKET_TARGET=4096 RBM_B1=9 timeout 300 python bench.py $B > $O/${LIB}_C5_t4096_b1_9.log 2>&1
RBM_BUCKET_TARGET=4096 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > $O/${LIB}_pytest.log 2>&1
done
unset RBM_LIB
grep -H '"value"' $O/*.log | python -c "
import sys, json
for l in sys.stdin:
    f, _, j = l.partition(':')
    try:
        d = json.loads(j)
        print(f.split('/')[-1], '%.3f ms' % d['ms_per_step'], '%.3e' % d['value'], d.get('kernel_ms_per_step'))
    except Exception as e:
        print(f, 'parse error', e)
" > $O/summary.txt 2>&1
echo done
