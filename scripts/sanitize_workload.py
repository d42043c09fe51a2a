"""Small workloads that reach every kernel of librbm.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck), one tool per run:

    compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_workload.py

Buckets are forced small (RBM_BUCKET_TARGET=64) so that N ~ 1e5 takes the
two-pass layout (prologue, split, bucket step with straddlers) the large
configurations use.  Plumbing only: everything runs in the library's kernels.
"""
import os
import sys

os.environ.setdefault("RBM_BUCKET_TARGET", "64")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import rbm_inputs as RI  # noqa: E402
from paper_1812_10575_b200 import RBM  # noqa: E402
from paper_1812_10575_b200 import partition as PT  # noqa: E402


def run(c, steps=3):
    s = RBM(c)
    s.run(steps)
    s.gather(host=True)
    s.close()


def main():
    run(RI.c5_coulomb_reg(n=100_003, p=2))                 # pair kernel, 2-pass, N odd (triple)
    run(RI.c5_coulomb_reg(n=100_000, p=8))                 # lane-group kernel
    run(dict(RI.c5_coulomb_reg(n=60_001, p=40)))           # one thread per batch (p > 32)
    run(RI.c4_aggregation(n=80_003))                       # keyed 16-B records, p = 4
    run(dict(RI.c2_sphere(n=50_000), integrator="split"))  # fp64 32-B records, split flow, sphere
    run(dict(RI.c4_aggregation(n=50_000), debug_bucket_cap=320))  # oversized buckets: global scratch
    run(RI.c1_dyson(n=500), steps=20)                      # resident kernel
    run(RI.c1_dyson(n=4000, scheme="rbmr"))                # RBM-r
    run(RI.c1_dyson(n=4000, scheme="rbmr_seq", integrator="split"))  # RBM-r'
    c = RI.cluster_sbm()
    run(c, steps=5)                                        # clustering model
    for fused in (False, True):                            # partitioned RBM-1 (loopback; fused = peer stores)
        ps = PT.PartitionedRBM(RI.c5_coulomb_reg(n=100_000, p=2), 2, range(2), PT.LoopbackExchange(fused=fused),
                               device="cuda:0")
        ps.run(3)
        ps.gather()
        ps.close()
    ps = PT.PartitionedRBM(dict(RI.c5_coulomb_reg(n=20_000, p=2), scheme="rbmr"), 2, range(2),
                           PT.LoopbackExchange(), device="cuda:0")
    ps.run(3)
    ps.gather()
    ps.close()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
