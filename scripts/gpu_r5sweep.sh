#!/bin/bash
# Layout sweep on the final kernels: mean bucket size (RBM_BUCKET_TARGET) and the
# pass-1 digit width (RBM_B1) at C5 (p = 2, 8) and C4.   usage: gpu_r5sweep.sh TAG
TAG=${1:-r5sweep}
O=gpurun_out/$TAG
mkdir -p $O
B="--steps 16 --warmup 3 --no-cpu-baseline --no-e2e"
for T in 2048 1536 1024 768 512; do
  RBM_BUCKET_TARGET=$T timeout 300 python bench.py $B > $O/C5_t$T.log 2>&1
  RBM_BUCKET_TARGET=$T timeout 300 python bench.py --workload C4 $B > $O/C4_t$T.log 2>&1
  RBM_BUCKET_TARGET=$T timeout 300 python bench.py --p 8 $B > $O/C5p8_t$T.log 2>&1
done
for B1 in 7 8 9 10; do
  RBM_B1=$B1 timeout 300 python bench.py $B > $O/C5_b1_$B1.log 2>&1
  RBM_B1=$B1 timeout 300 python bench.py --workload C4 $B > $O/C4_b1_$B1.log 2>&1
done
for T in 1024; do for B1 in 8 9 10; do
  RBM_BUCKET_TARGET=$T RBM_B1=$B1 timeout 300 python bench.py $B > $O/C5_t${T}_b1_$B1.log 2>&1
  RBM_BUCKET_TARGET=$T RBM_B1=$B1 timeout 300 python bench.py --workload C4 $B > $O/C4_t${T}_b1_$B1.log 2>&1
done; done
# 128-thread bucket CTAs (build.py -DRBM_BUCKET_BLOCK=128 -DRBM_BUCKET_ITEMS=10 -o librbm_b128.so): capacity <= 1280
export RBM_LIB=$PWD/paper_1812_10575_b200/librbm_b128.so
if [ -f $RBM_LIB ]; then
for T in 1024 768 512; do
  RBM_BUCKET_TARGET=$T timeout 300 python bench.py $B > $O/b128_C5_t$T.log 2>&1
  RBM_BUCKET_TARGET=$T RBM_B1=8 timeout 300 python bench.py $B > $O/b128_C5_t${T}_b1_8.log 2>&1
  RBM_BUCKET_TARGET=$T timeout 300 python bench.py --workload C4 $B > $O/b128_C4_t$T.log 2>&1
  RBM_BUCKET_TARGET=$T timeout 300 python bench.py --p 8 $B > $O/b128_C5p8_t$T.log 2>&1
done
RBM_BUCKET_TARGET=1024 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "one_step or permutation" > $O/b128_pytest.log 2>&1
fi
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
