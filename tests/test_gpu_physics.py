"""Long-run checks of the CUDA path (-m gpu): the GPU reaches what the paper
and the mathematics fix, and agrees with the oracle beyond one step.

  * Dyson, split integrator (D:16/17): the semicircle after T=10,
    and the GPU trajectory stays on the oracle's (contractive pair flow).
  * Thomson on S^2 (Sec. 5.1): annealed p=2 RBM then a p=N polish
    lands on the closed-form minima (octahedron, icosahedron).
  * Opinion dynamics C3 (D:18): same consensus-cluster count as the oracle
    at N=10^4 (T=5 and T=25) and the same empirical law (KS distance).
  * RBM-r (D:8): the Dyson second-moment trajectory matches RBM-1's and the
    closed form m2(t).
"""
import math

import numpy as np
import pytest

import rbm_inputs as RI
from test_oracle_pins import semicircle_cdf, thomson_energy, thomson_minimum, w1_to_cdf

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


@pytest.mark.parametrize("seed", [1, 2])
def test_gpu_dyson_split_semicircle_and_trajectory(R, O, seed):
    cfg = RI.c1_dyson(n=500, integrator="split", seed=seed)
    s = R.RBM(cfg)
    x0 = s.gather(host=True)
    s.run(10000)
    g = s.gather(host=True)
    s.close()
    assert w1_to_cdf(g.ravel(), semicircle_cdf) < 0.02
    o = O.run(cfg, x0, 0, 10000)
    assert E(g, o) <= 1e-9


@pytest.mark.parametrize("n", [6, 12])
def test_gpu_thomson_reaches_minimum(R, n):
    cfg = RI.c2_sphere(n=n, seed=n)
    s = R.RBM(cfg)
    x = s.gather(host=True)
    s.close()
    m = 0
    for dt, T in [(1e-2, 60.0), (3e-3, 60.0), (1e-3, 60.0)]:
        k = int(round(T / dt))
        s = R.RBM(dict(cfg, dt=dt, step0=m), x0=x)
        s.run(k)
        x = s.gather(host=True)
        s.close()
        m += k
    assert np.allclose(np.linalg.norm(x, axis=1), 1.0, atol=1e-12)
    emin = thomson_minimum(n)
    assert (thomson_energy(x) - emin) / emin < 2e-3
    s = R.RBM(dict(cfg, p=n, dt=5e-2, step0=m), x0=x)
    s.run(20000)
    x = s.gather(host=True)
    s.close()
    assert abs(thomson_energy(x) - emin) / emin < 1e-8


def clusters(x, gap=0.5, min_frac=1e-3):
    """Consensus clusters (D:18): sorted opinions split where the gap > 0.5;
    clusters with at least 0.1% of the particles."""
    s = np.sort(np.asarray(x, np.float64).ravel())
    cuts = np.flatnonzero(np.diff(s) > gap)
    sizes = np.diff(np.concatenate([[0], cuts + 1, [s.size]]))
    return int(np.sum(sizes >= min_frac * s.size))


def ks(a, b):
    a, b = np.sort(np.ravel(a)), np.sort(np.ravel(b))
    g = np.concatenate([a, b])
    return float(np.max(np.abs(np.searchsorted(a, g, "right") / a.size - np.searchsorted(b, g, "right") / b.size)))


@pytest.mark.parametrize("steps", [500, 2500])
def test_gpu_opinion_cluster_count_vs_oracle(R, O, steps):
    cfg = RI.c3_opinion(n=10_000, seed=4)
    s = R.RBM(cfg)
    x0 = s.gather(host=True)
    s.run(steps)
    g = s.gather(host=True)
    s.close()
    o = O.run(cfg, x0.astype(np.float64), 0, steps)
    assert clusters(g) == clusters(o)
    assert ks(g, o) < 0.01
    if steps == 2500:   # T=25: the paper's clustering regime (3-4 clusters)
        assert 2 <= clusters(g) <= 6


def test_gpu_rbmr_second_moment_matches_rbm1(R):
    n, steps = 2000, 1000
    c1 = RI.c1_dyson(n=n, integrator="split", seed=5)
    cr = dict(c1, scheme="rbmr")
    m2 = {}
    for name, c in (("rbm1", c1), ("rbmr", cr)):
        s = R.RBM(c)
        x0 = s.gather(host=True)
        s.run(steps)
        m2[name] = float((s.gather(host=True) ** 2).mean())
        m20 = float((x0 ** 2).mean())
        s.close()
    s2 = c1["sigma"] ** 2
    pred = (1 + s2) / 2 + (m20 - (1 + s2) / 2) * math.exp(-2.0)
    assert abs(m2["rbm1"] - pred) < 0.02
    assert abs(m2["rbmr"] - pred) < 0.02
    assert abs(m2["rbmr"] - m2["rbm1"]) < 0.02
