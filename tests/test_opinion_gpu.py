"""The paper's stochastic opinion dynamics (Sec. 5.2.2, PAPER.md:1197-1230;
row f4): closed window phi = chi_[0,1], alpha = 40, tau = 1e-4, N = 1e3, with
and without eps_N = N^{-1/3}, -m gpu.  Parity with the oracle on a lattice
where many partners sit exactly at the window edge |z| = 1 (closed: they
interact), and the oracle's consensus clusters after 5000 steps."""
import numpy as np
import pytest

import rbm_inputs as RI
from test_gpu_physics import clusters, ks

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


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_closed_window_parity_on_edge_lattice(R, O, dtype):
    n = 4000
    c = dict(RI.opinion_paper(n=n, dtype=dtype), init="user", step0=1)
    x0 = (np.arange(n) % 21).astype(np.float64).reshape(n, 1) * 0.5 - 5.0  # spacing 0.5: |z| = 1 often
    s = R.RBM(c, x0=x0)
    s.step()
    g = s.gather(host=True)
    o = O.rbm1_step(c, x0, 1)
    assert E(g, o) <= (1e-12 if dtype == "f64" else 1e-4)
    # the strict window gives a different map on this lattice
    st = O.rbm1_step(dict(c, kparam=[40.0, 1.0, 0.0]), x0, 1)
    assert np.max(np.abs(st - o)) > 1e-3
    s.close()


@pytest.mark.parametrize("noise", [False, True])
def test_paper_opinion_clusters_vs_oracle(R, O, noise):
    c = RI.opinion_paper(n=1000, noise=noise, seed=3)
    s = R.RBM(c)
    x0 = s.gather(host=True)
    s.run(5000)
    g = s.gather(host=True)
    s.close()
    o = O.run(c, x0, 0, 5000)
    assert clusters(g) == clusters(o)
    assert ks(g, o) < 0.05
