"""Direct O(N^2) step on the GPU and the paper's
convergence study of RBM-1 against it (Sec. 4.1, Theorem 3.1), -m gpu.

  * one direct step == oracle_direct_step (fp64 1e-12, fp32 1e-4), ragged N;
  * RBM with p = N == the direct step (the p = N special case of Eq. 2.2);
  * Theorem 3.1 / Fig. errdepN: the error of RBM-1 (p=2)
    against the fully coupled forward-Euler solution (tau = 2^-15) at T = 1
    decays like sqrt(tau) for the smooth test system, and is insensitive to N.
"""
import math

import numpy as np
import pytest

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


def E(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


def model(kernel, d, n, dtype="f64", **kw):
    kp = {"bounded_confidence": [1.0, 1.0], "coulomb_reg": [0.01]}.get(kernel, [])
    c = dict(d=d, n=n, p=2, dtype=dtype, scheme="rbm1", integrator="em", kernel=kernel, kparam=kp,
             potential="harmonic", vparam=[1.0], constraint="none", sigma=0.1, dt=1e-3, seed=77,
             init="normal", iparam=[0.0, 1.0])
    c.update(kw)
    return c


CASES = [("smooth", 1), ("gauss_attr_rep", 2), ("coulomb_reg", 3), ("bounded_confidence", 1),
         ("dyson", 1), ("zero", 3)]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kernel,d", CASES)
def test_direct_step_vs_oracle(R, O, kernel, d, dtype):
    n = 1001  # ragged against the 128-particle tiles
    c = model(kernel, d, n, dtype, step0=5)
    x0 = RI.user_x0(n, d, seed=11).astype(np.float32 if dtype == "f32" else np.float64)
    s = R.Direct(c, x0)
    s.run(1)
    g = s.gather()
    o = O.direct_step(c, x0.astype(np.float64), 5)
    if dtype == "f64":
        assert E(g, o) <= 1e-12
    elif kernel == "dyson":
        err = np.max(np.abs(g - o), axis=1) / max(1.0, np.max(np.abs(o)))
        assert np.quantile(err, 0.999) <= 1e-4
    else:
        assert E(g, o) <= 1e-4


def test_direct_sphere_vs_oracle(R, O):
    c = RI.c2_sphere(n=777, seed=3)
    x0 = RI.user_x0(777, 3, seed=3, dist="sphere")
    s = R.Direct(c, x0)
    s.run(1)
    g = s.gather()
    assert E(g, O.direct_step(c, x0, 0)) <= 1e-12
    assert np.max(np.abs(np.linalg.norm(g, axis=1) - 1.0)) < 1e-14


def test_direct_many_steps_vs_oracle(R, O):
    c = model("smooth", 1, 600)
    x0 = RI.user_x0(600, 1, seed=2)
    s = R.Direct(c, x0)
    s.run(50)
    assert E(s.gather(), O.run(dict(c, p=600), x0, 0, 50)) <= 1e-9


def test_rbm_p_equals_n_is_direct(R):
    n = 1500
    c = model("gauss_attr_rep", 2, n, p=n)
    x0 = RI.user_x0(n, 2, seed=9)
    s = R.RBM(c, x0=x0)
    s.run(20)
    a = s.gather(host=True)
    s.close()
    d = R.Direct(c, x0)
    d.run(20)
    assert E(a, d.gather()) <= 1e-12


def smooth_system(n, beta, seed):
    return dict(RI.smooth_test(n, p=2, beta=beta, seed=seed), sigma=0.0, init="user")


def rbm_error(R, n, beta, tau_exp, T=1.0, seed=1, ref=None):
    """E^(T) of Eq. (4.2): RBM-1 p=2 with tau = 2^-tau_exp vs the
    fully coupled forward Euler solution with tau = 2^-15, same X_0."""
    x0 = RI.semicircle_x0(n, seed=seed)
    cfg = smooth_system(n, beta, seed)
    if ref is None:
        d = R.Direct(dict(cfg, dt=2.0 ** -15), x0)
        d.run(int(round(T * 2 ** 15)))
        ref = d.gather()
    s = R.RBM(dict(cfg, dt=2.0 ** -tau_exp), x0=x0)
    s.run(int(round(T * 2 ** tau_exp)))
    x = s.gather(host=True)
    s.close()
    return float(np.sqrt(np.mean((x - ref) ** 2))), ref


def test_convergence_half_order_in_tau(R):
    """Fig. errdepN: log E^ vs log tau has slope ~0.5 (N = 2000, beta = 1)."""
    errs, ref = [], None
    exps = [4, 5, 6, 7]
    for k in exps:
        e, ref = rbm_error(R, 2000, 1.0, k, ref=ref)
        errs.append(e)
    # average over three division seeds (one run per seed, as the paper)
    slope = np.polyfit(np.log([2.0 ** -k for k in exps]), np.log(errs), 1)[0]
    assert 0.3 <= slope <= 0.75, (slope, errs)
    assert errs[-1] < errs[0]


def test_convergence_insensitive_to_n(R):
    """Fig. errdepN: the error at fixed tau barely depends on N (500 vs 2000)."""
    e500, _ = rbm_error(R, 500, 1.0, 6, seed=4)
    e2000, _ = rbm_error(R, 2000, 1.0, 6, seed=4)
    assert 0.5 <= e500 / e2000 <= 2.0, (e500, e2000)
