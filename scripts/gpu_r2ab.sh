#!/bin/bash
# L2 fetch granularity (cudaLimitMaxL2FetchGranularity) for the random-access kernels
mkdir -p gpurun_out/r2ab
O=gpurun_out/r2ab
python - > $O/limit.txt 2>&1 <<'PY'
import ctypes
import torch; torch.cuda.init()
try:
    rt = ctypes.CDLL("libcudart.so.12")
except OSError:
    rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
v = ctypes.c_size_t(0)
print("default MaxL2FetchGranularity rc", rt.cudaDeviceGetLimit(ctypes.byref(v), 0x05), v.value)
PY
for G in 32 64 128; do
for S in rbmr rbmr_seq; do
RBM_L2_FETCH=$G timeout -s KILL 300 python bench.py --scheme $S --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > $O/${S}_$G.log 2>&1
done
RBM_L2_FETCH=$G timeout -s KILL 300 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > $O/rbm1_$G.log 2>&1
done
CMD="python bench.py --scheme rbmr_seq --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
RBM_L2_FETCH=32 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/launches_seq32.csv $CMD > $O/ncu_seq32.log 2>&1
