"""Long-run fp32 statistics of C4 and C5 against the oracle (-m gpu).

BASELINE.json north_star: "fp32 mode is checked at 1e-4 after 1 step and
statistically (equilibrium histograms and energies within stated confidence
bands) on long runs".  C4 and C5 have no closed-form equilibrium (SURVEY
8(c.10) last row), so the reference is the oracle's own long run from the
same X_0 and seed (same divisions, same Brownian increments; the oracle works
in IEEE double).  The trajectories separate only through rounding amplified at
close encounters, so the stated bands are far tighter than the two-sample KS
critical values for independent samples (1.36 sqrt(2/N) = 0.0061 at 95%,
N = 10^5), and any real error in the step -- a dropped term, a wrong sign,
a wrong batch -- moves these statistics by orders of magnitude more.
"""
import numpy as np
import pytest
from scipy import stats

import rbm_inputs as RI

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1812_10575_b200 import rbm
    rbm.lib()
    return rbm


def _run_both(R, O, cfg, steps):
    s = R.RBM(cfg)
    x0 = s.gather(host=True).astype(np.float64)
    s.run(steps)
    g = s.gather(host=True).astype(np.float64)
    s.close()
    o = O.run(cfg, x0, 0, steps)
    return x0, g, o


def test_c5_long_run_statistics(R, O):
    """C5 physics (regularised Coulomb, harmonic V, sigma 0.1, fp32) at N = 10^5,
    p = 2, 2000 steps (T = 2): second moment within 1e-3 relative, radial
    distribution KS distance < 0.005, mean position within 1e-3."""
    c = RI.c5_coulomb_reg(n=100_000, p=2)
    x0, g, o = _run_both(R, O, c, 2000)
    m2g, m2o = float(np.mean(np.sum(g * g, 1))), float(np.mean(np.sum(o * o, 1)))
    m20 = float(np.mean(np.sum(x0 * x0, 1)))
    ks = stats.ks_2samp(np.linalg.norm(g, axis=1), np.linalg.norm(o, axis=1)).statistic
    print(f"C5 long run: m2 {m20:.5f} -> gpu {m2g:.6f} oracle {m2o:.6f}; radial KS {ks:.2e}")
    assert abs(m2g / m2o - 1.0) < 1e-3
    assert abs(m2g - m20) > 0.1            # the run moved the system (harmonic contraction)
    assert ks < 0.005
    assert np.max(np.abs(g.mean(0) - o.mean(0))) < 1e-3


def test_c4_long_run_histograms(R, O):
    """C4 physics (Gaussian attraction-repulsion, 5-Gaussian mixture, fp32) at
    N = 10^5, p = 4, the configured 100 steps: per-axis histogram KS < 0.005
    and the second moment within 1e-3 relative."""
    c = RI.c4_aggregation(n=100_000)
    x0, g, o = _run_both(R, O, c, 100)
    for a in range(2):
        ks = stats.ks_2samp(g[:, a], o[:, a]).statistic
        print(f"C4 axis {a}: KS {ks:.2e}")
        assert ks < 0.005
    m2g, m2o = float(np.mean(np.sum(g * g, 1))), float(np.mean(np.sum(o * o, 1)))
    assert abs(m2g / m2o - 1.0) < 1e-3
    # the aggregation moved the system: the histograms differ from X_0's
    assert stats.ks_2samp(g[:, 0], x0[:, 0]).statistic > 0.02
