"""C1 (N=500, resident kernel) timing diagnostic: rbm_run(K) with and without
the per-kernel event timing, CUDA events on the library's stream."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import rbm_inputs as RI
from paper_1812_10575_b200 import RBM
s = RBM(RI.c1_dyson())
st = s.stream
s.run(50); s.sync()
for K in (100, 1000, 1000, 4000):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st); s.run(K); e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"K={K} run: {ms:.3f} ms  {ms*1e3/K:.2f} us/step  {500*K/ms*1e3:.3e} particle-steps/s")
s.timing_begin(1000)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record(st); s.run(1000); e1.record(st); torch.cuda.synchronize()
pk, n = s.timing_end()
print("timed run:", e0.elapsed_time(e1), "per-kernel", pk, n)
