"""RBM-r at layouts with B = 19..20 (ids per bucket via RBM_RBMR_W): run 2 steps, report errors."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(1 << 26, 128), (1 << 27, 128), (1 << 28, 256), ((1 << 20) + 7, 128)]
if len(sys.argv) > 1 and sys.argv[1] == "one":
    sys.path.insert(0, ROOT)
    import numpy as np
    import rbm_inputs as RI
    from paper_1812_10575_b200 import RBM
    n = int(sys.argv[2])
    c = RI.c5_coulomb_reg(n=n, scheme="rbmr")
    s = RBM(c)
    print("layout", s.layout, flush=True)
    s.step()
    s.sync()
    s.step()
    s.sync()
    g = s.gather(0, 1000, host=True)
    print("ok", np.isfinite(g).all(), flush=True)
    sys.exit(0)
for n, w in CASES:
    for lib in ("librbm.so", "librbm_checked.so"):
        env = dict(os.environ, RBM_RBMR_W=str(w), RBM_LIB=os.path.join(ROOT, "paper_1812_10575_b200", lib))
        r = subprocess.run([sys.executable, __file__, "one", str(n)], env=env, capture_output=True, text=True, timeout=300)
        print(n, w, lib, "rc", r.returncode, r.stdout.strip()[-300:], r.stderr.strip()[-400:], flush=True)
