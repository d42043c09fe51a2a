"""Wealth model (Sec. 5.2.1) on the
GPU, -m gpu: parity with the oracle (split with the exact linear pair flow and
the exact geometric-Brownian-motion noise step; Euler-Maruyama with
multiplicative noise) and the paper's equilibrium, the inverse-Gamma law
(shape kappa/D + 1 = 2, scale kappa eta/D, eta = sqrt(2/pi) the mean wealth)."""
import math

import numpy as np
import pytest

import rbm_inputs as RI
from test_oracle_pins import inv_gamma2_cdf

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1812_10575_b200 import rbm
    rbm.lib()
    return rbm


def E(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


@pytest.mark.parametrize("n", [1000, 100_000, 3_000_000])
@pytest.mark.parametrize("integrator", ["split", "em"])
def test_wealth_one_step_parity(R, O, n, integrator):
    c = dict(RI.wealth(n=n, integrator=integrator, seed=3), step0=4)
    s = R.RBM(c)
    x0 = s.gather(host=True)
    assert E(x0, O.init(c)) <= 1e-14  # both fp64; libm vs CUDA log/sincospi differ by ulps
    s.step()
    assert E(s.gather(host=True), O.rbm1_step(c, x0, 4)) <= 1e-12
    s.close()


def test_wealth_100_steps_parity_and_fp32(R, O):
    c = RI.wealth(n=20_000, seed=5)
    s = R.RBM(c)
    x0 = s.gather(host=True)
    s.run(100)
    assert E(s.gather(host=True), O.run(c, x0, 0, 100)) <= 1e-9
    s.close()
    c32 = dict(c, dtype="f32")
    s = R.RBM(c32)
    x0 = s.gather(host=True).astype(np.float64)
    s.step()
    assert E(s.gather(host=True), O.rbm1_step(c32, x0, 0)) <= 1e-4
    s.close()


def test_wealth_gpu_reaches_inverse_gamma(R):
    """Fig. wealth: N = 1e5 agents, tau = 1e-3, T = 3."""
    c = RI.wealth(n=100_000, seed=7)
    s = R.RBM(c)
    x0 = s.gather(host=True).ravel()
    eta = math.sqrt(2.0 / math.pi)
    s.run(3000)
    x = s.gather(host=True).ravel()
    s.close()
    assert np.all(x > 0)
    srt = np.sort(x)
    ks = np.max(np.abs(np.arange(1, srt.size + 1) / srt.size - inv_gamma2_cdf(srt, eta)))
    assert ks < 0.015, ks
    # the splitting keeps the mean wealth in expectation
    assert abs(x.mean() - x0.mean()) < 0.05 * eta


def test_wealth_partitioned_bit_identical(R):
    from paper_1812_10575_b200 import partition as PT
    c = RI.wealth(n=200_000, seed=9)
    s = R.RBM(c)
    s.run(7)
    a = s.gather(host=True)
    s.close()
    ps = PT.PartitionedRBM(c, 4, range(4), PT.LoopbackExchange(fused=True))
    ps.run(7)
    b = ps.gather().cpu().numpy()
    ps.close()
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
