"""Memory-safety tier (-m gpu): the kernels' index bounds asserted.

compute-sanitizer is closed on this GPU pool (tests/test_sanitizer.py), so
librbm_checked.so -- the same library built with -DRBM_CHECKED=1, where every
shared-memory staging index, sort rank, staged output slot, straddler member
slot and RBM-r increment index is checked against its bound and a violation
sets the device flag reported as RBM_ERR_CAPACITY ("bounds check") -- runs the
workload that reaches every kernel (scripts/sanitize_workload.py: forced small
buckets so N ~ 1e5 takes the 2-pass layout, oversized buckets, p = 2 / 4 / 8 /
40, fp32 and fp64, split flows, sphere, resident kernel, RBM-r, RBM-r',
clustering, partitioned RBM-1 with and without peer stores, partitioned RBM-r).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1812_10575_b200", "librbm_checked.so")


def test_checked_build_clean_on_every_kernel():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    assert os.path.exists(LIB), "librbm_checked.so not built (__graft_entry__.build)"
    env = dict(os.environ, RBM_LIB=LIB)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_workload.py")],
                       capture_output=True, text=True, timeout=1200, env=env)
    log = r.stdout + r.stderr
    assert r.returncode == 0, log[-4000:]
    assert "sanitize workload done" in log
