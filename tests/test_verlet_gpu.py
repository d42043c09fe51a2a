"""Second-order RBM with Verlet (PAPER.md:848-878,
Appendix A) on the GPU, -m gpu: parity with the oracle (start step and
position form), checkpoint/resume in the (x_n, x_{n-1}) form, the full-force
Verlet reference (direct step), and Fig. second: the RBM-1 error against the
full-force solution at T = 1 decays like sqrt(tau)."""
import numpy as np
import pytest

import rbm_inputs as RI
from test_oracle_pins import verlet_cfg

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


def xv0(n, seed):
    rng = np.random.default_rng(seed)
    return np.stack([RI.semicircle_x0(n, seed=seed).ravel(), rng.standard_normal(n)], axis=1)


@pytest.mark.parametrize("n,p", [(1000, 2), (50_001, 2), (50_001, 5), (3_000_001, 2)])
def test_verlet_steps_vs_oracle(R, O, n, p):
    c = verlet_cfg(n, p=p, seed=3)
    x0 = xv0(n, 3)
    s = R.RBM(c, x0=x0)
    s.step()                      # start step from (x_0, v_0)
    assert E(s.gather(host=True), O.rbm1_step(c, x0, 0)) <= 1e-12
    s.run(9)                      # position form
    assert E(s.gather(host=True), O.run(c, x0, 0, 10)) <= 1e-10
    s.close()


def test_verlet_resume_in_position_form(R):
    c = verlet_cfg(40_000, p=2, seed=5)
    x0 = xv0(40_000, 5)
    a = R.RBM(c, x0=x0)
    a.run(20)
    full = a.gather(host=True)
    a.close()
    b = R.RBM(c, x0=x0)
    b.run(8)
    mid = b.gather(host=True)
    b.close()
    r = R.RBM(dict(c, state_form="xx", step0=8), x0=mid)
    r.run(12)
    assert np.array_equal(r.gather(host=True), full)
    r.close()


def test_verlet_direct_vs_oracle(R, O):
    c = verlet_cfg(700, p=2)
    x0 = xv0(700, 2)
    d = R.Direct(c, x0)
    d.run(25)
    assert E(d.gather(), O.direct_run(c, x0, 0, 25)) <= 1e-11


def test_verlet_direct_chunked_runs_compose(R):
    """run(10) then run(15) == run(25): the Verlet start formula
    applies to the first step of the whole run only."""
    c = verlet_cfg(700, p=2)
    x0 = xv0(700, 3)
    a = R.Direct(c, x0)
    a.run(25)
    b = R.Direct(c, x0)
    b.run(10)
    b.run(15)
    assert np.array_equal(a.gather(), b.gather())


def test_verlet_convergence_half_order(R):
    """Fig. second: N = 500, T = 1, reference tau = 2^-15 (full force), RBM-1 p=2."""
    n = 500
    x0 = xv0(n, 9)
    d = R.Direct(verlet_cfg(n, dt=2.0 ** -15), x0)
    d.run(2 ** 15)
    ref = d.gather()
    errs = []
    exps = [4, 5, 6, 7]
    for k in exps:
        s = R.RBM(verlet_cfg(n, dt=2.0 ** -k, seed=13), x0=x0)
        s.run(2 ** k)
        y = s.gather(host=True)
        s.close()
        errs.append(float(np.sqrt(np.mean((y[:, 0] - ref[:, 0]) ** 2))))
    slope = np.polyfit(np.log([2.0 ** -k for k in exps]), np.log(errs), 1)[0]
    assert 0.3 <= slope <= 0.8, (slope, errs)
