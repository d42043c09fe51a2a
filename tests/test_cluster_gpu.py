"""Clustering through the interacting particle system (Sec. 5.3, PAPER.md
1240-1300) on the GPU (-m gpu).

The picked pair (i, j) follows dX^i/dt = alpha (a_ij - beta)(X^j - X^i)
(P:1252), solved exactly by the update formula of P:1258-1264; a_ij from a CSR
adjacency; RBM-r with p = 2 (Jacobi sweep, reading D:8) and the sequential
RBM-r'.  Parity against the oracle, then the paper's SBM experiment (reading
D:26: 2-D positions, recovery by 3-means of the whitened positions).
"""
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
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


@pytest.mark.parametrize("scheme", ["rbmr", "rbmr_seq"])
@pytest.mark.parametrize("edges", [False, True])
@pytest.mark.parametrize("d", [1, 2])
def test_cluster_parity(R, O, scheme, edges, d):
    c = dict(RI.cluster_sbm(d=d, seed=4, edge_restricted=edges, scheme=scheme), step0=2)
    s = R.RBM(c)
    x0 = s.gather(host=True)
    s.step()
    assert np.array_equal(s.slots(), O.rbmr_slots(c, 2))
    one = O.rbmr_step(c, x0, 2) if scheme == "rbmr" else O.rbmr_seq_step(c, x0, 2)
    assert E(s.gather(host=True), one) <= 1e-12
    s.run(100)
    ref = O.run(c, one, 3, 100)
    assert E(s.gather(host=True), ref) <= 1e-9
    s.close()


def test_cluster_needs_adjacency(R):
    c = RI.cluster_sbm()
    c.pop("adjacency")
    s = R.RBM(c)
    with pytest.raises(R.RbmError) as e:
        s.step()
    assert e.value.status == 8
    s.close()


@pytest.mark.parametrize("seed", [1, 3, 5])
def test_sbm_recovery(R, seed):
    """N = 1200 (200/400/600), p = 0.7, q = 0.3, alpha = 40, beta = 1/2,
    tau = 1e-3, X_0 ~ U[0, 50]^2, T = 5: the blocks are recovered (ARI >= 0.95)."""
    from sklearn.cluster import KMeans
    from sklearn.metrics import adjusted_rand_score
    c = RI.cluster_sbm(seed=seed)
    s = R.RBM(c)
    s.run(c["steps"])
    x = s.gather(host=True)
    s.close()
    z = x - x.mean(0)
    w = np.linalg.cholesky(np.linalg.inv(np.cov(z.T)))
    lab = KMeans(3, n_init=10, random_state=0).fit(z @ w).labels_
    ari = adjusted_rand_score(c["labels"], lab)
    print(f"SBM seed {seed}: ARI {ari:.4f}")
    assert ari >= 0.95
